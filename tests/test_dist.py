"""CPU, world_size 2 over gloo: the product's sharding and reduction code (SURVEY §8.1 row e).

The device kernels need a GPU (test_gpu_dist.py runs the sharded conv itself on one device); here the
product's host side runs under a real 2-rank process group:
* ``partition_by_cost`` / ``shard`` (batch elements) and ``leaf_aligned_ranges`` (output rows of one grid)
  cover the work exactly once and balance it;
* ``WgradReducer`` (the in-backward asynchronous all-reduce) and ``allreduce_gradients`` (flattened
  multi-tensor path, gradient tensors or Parameters) sum the per-rank weight gradients.
Per-rank gradients are computed by a float64 torch evaluation of C6 over the oracle's kernel-map table
restricted to the rank's share, and the sum must equal the full-batch / full-grid gradient.
"""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2407_01781_b200.dist import (WgradReducer, allreduce_gradients, leaf_aligned_ranges, partition_by_cost,
                                        shard)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    rng = np.random.default_rng(0)
    grids = [O.build_from_coords(rng.integers(-s, s, size=(n, 3))) for s, n in ((6, 80), (9, 200), (5, 60), (8, 150))]
    maps = [O.kernel_map(g, g, 1) for g in grids]
    w = rng.normal(size=(3, 4, 3, 3, 3))
    feats = [rng.normal(size=(g.num_voxels, 4)) for g in grids]
    gos = [rng.normal(size=(g.num_voxels, 3)) for g in grids]
    return grids, maps, w, feats, gos


def _wgrad_rows(table, x, go, rows):
    """float64 C6 wgrad over output rows ``rows`` of a [27, n] table: gw[co, ci, d] = sum go[o,co] x[t[d,o],ci]."""
    t = torch.from_numpy(table[:, rows])
    xs, gs = torch.from_numpy(x), torch.from_numpy(go[rows])
    gw = torch.zeros(gs.shape[1], xs.shape[1], 27, dtype=torch.float64)
    for d in range(27):
        m = t[d] >= 0
        gw[:, :, d] = gs[m].T @ xs[t[d][m]]
    return gw.reshape(gs.shape[1], xs.shape[1], 3, 3, 3)


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    grids, maps, w, feats, gos = _problem()
    res = {}
    # batch sharding by pairs + the asynchronous reducer
    costs = [sum(len(o) for o in m[1]) for m in maps]
    gw = torch.zeros(w.shape, dtype=torch.float64)
    for b in shard(list(range(len(grids))), rank, world, costs):
        table = O.kernel_map_table(*maps[b], grids[b].num_voxels)
        gw += _wgrad_rows(table, feats[b], gos[b], slice(0, grids[b].num_voxels))
    red = WgradReducer()
    h = red.start(gw)
    red.wait(h)
    res["batch"] = gw.numpy()
    # row sharding of the largest grid at leaf boundaries + the flattened multi-tensor all-reduce
    g, m = grids[1], maps[1]
    table = O.kernel_map_table(*m, g.num_voxels)
    r0, r1, _, _ = leaf_aligned_ranges(g.leaf_value_offset, g.num_voxels, world)[rank]
    p1 = torch.nn.Parameter(torch.zeros(w.shape, dtype=torch.float64))
    p1.grad = _wgrad_rows(table, feats[1], gos[1], slice(r0, r1))
    g2 = torch.full((5,), float(rank + 1), dtype=torch.float64)  # a gradient tensor passed directly
    allreduce_gradients([p1, g2])
    res["rows"] = p1.grad.numpy()
    res["g2"] = g2.numpy()
    out_q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_and_reduction_equal_full_problem():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    grids, maps, w, feats, gos = _problem()
    full = sum(O.conv_backward(m[0], m[1], go, f, w)[1] for m, go, f in zip(maps, gos, feats))
    full_rows = O.conv_backward(maps[1][0], maps[1][1], gos[1], feats[1], w)[1]
    for r in range(2):
        assert np.allclose(res[r]["batch"], full, rtol=1e-12, atol=1e-12)
        assert np.allclose(res[r]["rows"], full_rows, rtol=1e-12, atol=1e-12)
        assert np.array_equal(res[r]["g2"], np.full(5, 3.0))
    assert np.array_equal(res[0]["batch"], res[1]["batch"])


def test_leaf_aligned_ranges_cover_rows_at_leaf_boundaries():
    rng = np.random.default_rng(2)
    g = O.build_from_coords(rng.integers(-40, 40, size=(3000, 3)))
    starts = set((np.asarray(g.leaf_value_offset, np.int64) - 1).tolist()) | {g.num_voxels}
    for world in (1, 2, 3, 8):
        rs = leaf_aligned_ranges(g.leaf_value_offset, g.num_voxels, world)
        assert rs[0][0] == 0 and rs[-1][1] == g.num_voxels
        for (a, b, l0, l1), (c, _, l2, _) in zip(rs, rs[1:]):
            assert b == c and l1 == l2
        assert all(r0 in starts and r1 in starts for r0, r1, _, _ in rs)
        sizes = [r1 - r0 for r0, r1, _, _ in rs]
        assert max(sizes) - min(sizes) <= 512  # balanced to within one leaf
