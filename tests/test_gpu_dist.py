"""GPU: the product's sharded paths (SURVEY §8.1 row e) on one device.

* Row shards (cfg5 sharding): R leaf-aligned RowShards computed one after another on one GPU must give the
  unsharded forward and input gradient row for row, bitwise (every output row sees the same neighbour
  entries in the same offset order), and weight-gradient partials that sum to the unsharded gradient.
* Batch shards (cfg3 sharding): each shard's batched kernel map / conv / wgrad, summed, equal the whole batch.
* The module's in-backward all-reduce under a real NCCL process group (world 1; the exchange is exercised,
  the sum is the identity) gives the same gradients as without it.
Multi-GPU runs (world > 1) are in test_gpu_dist_nccl below and skip on one device.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import paper_2407_01781_b200 as P
from paper_2407_01781_b200 import dist as D
from paper_2407_01781_b200.conv import gather_conv, wgrad
from paper_2407_01781_b200.workloads import lidar_scan_points, sphere_shell_coords

pytestmark = pytest.mark.gpu


def _shell(res=96):
    g, _ = P.build_from_coords(sphere_shell_coords(res, band=1.5))
    return g


@pytest.mark.parametrize("dtype,impl", [(torch.float32, None), (torch.bfloat16, "gather"), (torch.bfloat16, "halo")])
@pytest.mark.parametrize("R", [2, 3, 8])
def test_row_shards_reassemble_the_full_conv(dtype, impl, R, monkeypatch):
    if impl:
        monkeypatch.setenv("FVDB_CONV_IMPL", impl)
    g = _shell()
    C = 32
    gen = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(g.num_voxels, C, device="cuda", generator=gen).to(dtype)
    gy = torch.randn(g.num_voxels, C, device="cuda", generator=gen).to(dtype)
    w = torch.randn(C, C, 3, 3, 3, device="cuda", generator=gen) / (27 * C) ** 0.5
    if dtype != torch.bfloat16:
        w = w.to(dtype)
    km = P.build_kernel_map(g, g, 1)
    y_full = gather_conv(x, km.fwd, w)
    gx_full = gather_conv(gy, km.bwd, w, transpose=True)
    gw_full = wgrad(x, gy, km.fwd)
    ranges = D.leaf_aligned_ranges(g.leaf_value_offset, g.num_voxels, R)
    assert ranges[0][0] == 0 and ranges[-1][1] == g.num_voxels
    ys, gxs, gw, pairs = [], [], torch.zeros_like(gw_full), 0
    for (r0, r1, l0, l1) in ranges:
        sh = D.RowShard(g, r0, r1, l0, l1)
        assert torch.equal(sh.fwd.view, km.nbr[:, r0:r1])  # the shard's map is the full map's columns
        ys.append(sh.forward(x, w))
        gxs.append(sh.input_grad(gy, w))
        gw += sh.weight_grad(x, gy[r0:r1]).to(gw.dtype)
        pairs += sh.total_pairs
    assert pairs == km.total_pairs
    assert torch.equal(torch.cat(ys), y_full)
    assert torch.equal(torch.cat(gxs), gx_full)
    rel = float((gw - gw_full).norm() / gw_full.norm())
    assert rel < 1e-5, rel


def test_batch_shards_sum_to_the_whole_batch():
    pts = [lidar_scan_points(s)[::4] for s in range(5)]
    batch, _ = P.build_from_points(P.jagged_from_list([torch.from_numpy(p) for p in pts]), P.VoxelTransform.uniform(0.05))
    km = P.build_batch_kernel_map(batch, batch, 1)
    C = 64
    gen = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(batch.total_voxels, C, device="cuda", generator=gen).to(torch.bfloat16)
    gy = torch.randn(batch.total_voxels, C, device="cuda", generator=gen).to(torch.bfloat16)
    w = torch.randn(C, C, 3, 3, 3, device="cuda", generator=gen) / (27 * C) ** 0.5
    gw_full = wgrad(x, gy, km.fwd)
    y_full = gather_conv(x, km.fwd, w)
    costs = [int(P.build_kernel_map(gr, gr, 1).total_pairs) for gr in batch.grids]
    for R in (2, 3):
        gw = torch.zeros_like(gw_full)
        ys = []
        for r in range(R):
            sub, (s, e) = D.shard_batch(batch, r, R, costs)
            if sub is None:
                continue
            rows = slice(int(batch.voxel_joffsets[s, 0]), int(batch.voxel_joffsets[e - 1, 1]))
            k = P.build_batch_kernel_map(sub, sub, 1)
            ys.append(gather_conv(x[rows], k.fwd, w))
            gw += wgrad(x[rows], gy[rows], k.fwd)
        assert torch.equal(torch.cat(ys), y_full)
        assert float((gw - gw_full).norm() / gw_full.norm()) < 1e-5


_WORLD1 = r"""
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.workloads import sphere_shell_coords
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
g, _ = P.build_from_coords(sphere_shell_coords(64, band=1.5))
m = P.SparseConv3d(32, 32).cuda()
x = torch.randn(g.num_voxels, 32, device="cuda", requires_grad=True)
gy = torch.randn(g.num_voxels, 32, device="cuda")
_, y = m(g, x)
y.jdata.backward(gy.to(y.jdata.dtype))
gw0, gx0 = m.weight.grad.clone(), x.grad.clone()
m.weight.grad = None; x.grad = None
r = P.dist.attach_grad_reducer(m)
_, y = m(g, x)
y.jdata.backward(gy.to(y.jdata.dtype))
assert r.calls == 1, r.calls
assert torch.equal(m.weight.grad, gw0) and torch.equal(x.grad, gx0)
dist.destroy_process_group()
print("OK")
"""


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_module_allreduce_in_backward_nccl_world1(tmp_path):
    f = tmp_path / "w1.py"
    f.write_text(_WORLD1)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0", WORLD_SIZE="1",
               LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(f)], cwd=str(__import__("pathlib").Path(__file__).parents[1]), env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("config", ["cfg3", "cfg2"])
def test_bench_torchrun_two_ranks(config):
    root = __import__("pathlib").Path(__file__).parents[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
                        "--steps", "3", "--warmup", "3", "--config", config, "--no-cpu-baseline", "--e2e-steps", "3"],
                       cwd=str(root), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    assert '"n_gpus": 2' in r.stdout
