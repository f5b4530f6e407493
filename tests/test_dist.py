"""CPU, world_size 2 over gloo: batch sharding + the wgrad sum all-reduce (SURVEY §8.1 row e).

Each rank computes the weight gradient of its shard of grids with the oracle (the
device kernels need a GPU; the exchange logic is what is under test here) and the
all-reduced result must equal the full-batch gradient — batched wgrad is the sum of
per-element wgrads.
"""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2407_01781_b200.dist import allreduce_gradients, partition_by_cost


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


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    grids, maps, w, feats, gos = _problem()
    costs = [sum(len(o) for o in m[1]) for m in maps]
    s, e = partition_by_cost(costs, world)[rank]
    gw = np.zeros_like(w)
    for b in range(s, e):
        ins, outs = maps[b]
        gw += O.conv_backward(ins, outs, gos[b], feats[b], w)[1]
    p = torch.nn.Parameter(torch.zeros(w.shape, dtype=torch.float64))
    p.grad = torch.from_numpy(gw)
    allreduce_gradients([p])
    out_q.put((rank, p.grad.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_wgrad_allreduce_equals_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    grids, maps, w, feats, gos = _problem()
    full = sum(O.conv_backward(m[0], m[1], go, f, w)[1] for m, go, f in zip(maps, gos, feats))
    for r in range(2):
        assert np.allclose(res[r], full, rtol=1e-12, atol=1e-12)
    assert np.array_equal(res[0], res[1])
