"""GPU: halo plan invariants and the halo-staged tensor-core conv (csrc/conv_halo.cu).

The halo kernel computes the reference operator (conv.py:180-191 forward, conv.py:358-366 dgrad
form); these tests pin it against the oracle on bf16-rounded inputs (accumulation error only,
rel ≤ 2e-5), against the gather-GEMM kernel, and check the plan itself exactly: every
(offset, lane) slot must resolve to the kernel map's input row.
"""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.conv import gather_conv
from paper_2407_01781_b200.workloads import sphere_shell_coords
from conftest import KMAP_CASES

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = a.detach().double().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def bf16_round(a):
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).float().numpy().astype(np.float64)


def check_plan(table, K, N):
    """Exact plan invariants: lane permutation, slot -> input row, masks, phase capacity."""
    plan = table.halo_plan(K, N)
    t = {k: v.cpu().numpy() for k, v in plan.tensors.items()}
    n, T = table.n, (table.n + 127) // 128
    nbr = table.view.cpu().numpy()
    perm = t["perm"].reshape(T, 128)
    valid = perm[perm >= 0]
    assert np.array_equal(np.sort(valid), np.arange(n)), "perm is not a permutation of the output rows"
    rec = t["tile_rec"].reshape(T, -1)
    lnbr = rec[:, :6912].copy().view(np.uint16).reshape(T, 27, 128).transpose(1, 0, 2).astype(np.int64)
    level = t["tile_level"]
    assert set(np.unique(level)) <= {1, 3, 9, 27}
    phase = t["phase"]
    hr = t["halo_rows"]
    masks = rec[:, 6912:6912 + 432].copy().view(np.uint32).reshape(T, 27, 4)
    # tiles' slot ranges are disjoint (single-pass plans allocate them by a device counter, in any order)
    ends = t["tile_base"] + np.array([max(int(phase[i, g, 0] + phase[i, g, 1]) for g in range(level[i]))
                                      for i in range(T)])
    order = np.argsort(t["tile_base"], kind="stable")
    assert np.all(t["tile_base"][order][1:] >= ends[order][:-1]), "tile slot ranges overlap"
    assert ends.max() <= hr.shape[0]
    rev = bool(plan.c.offsets_reversed)  # the forward plan run on the reversed (transposed) table
    for tile in range(T):
        gs = 27 // level[tile]
        for d in range(27):
            rd = 26 - d if rev else d
            g = rd // gs
            off, cnt = phase[tile, g]
            assert cnt <= plan.cap and cnt % 8 == 0
            lanes = np.arange(128)
            o = perm[tile]
            want = np.where(o >= 0, nbr[d][np.maximum(o, 0)], -1)
            s = lnbr[rd, tile]
            has = s != 0xFFFF
            assert np.array_equal(has, want >= 0), (tile, d)
            assert np.all(s[has] < cnt)
            got = hr[t["tile_base"][tile] + off + s[has]]
            assert np.array_equal(got, want[has]), (tile, d)
            bits = np.zeros(128, bool)
            for wd in range(4):
                bits[32 * wd:32 * wd + 32] = (masks[tile, rd, wd] >> np.arange(32, dtype=np.uint32)) & 1
            assert np.array_equal(bits, ~has), (tile, d)
            del lanes
    return plan


@pytest.mark.parametrize("name", KMAP_CASES)
@pytest.mark.parametrize("stride", [1, 2])
def test_halo_plan_exact(golden_grids, name, stride):
    c = golden_grids[f"{name}/coords"]
    g, _ = P.build_from_coords(c)
    go = g if stride == 1 else P.coarsen(g, 2)
    km = P.build_kernel_map(g, go, stride)
    check_plan(km.fwd, 64, 64)
    check_plan(km.bwd, 64, 64)
    check_plan(km.fwd, 128, 128)


def dense_cube(n=16):
    r = np.arange(n)
    return np.stack(np.meshgrid(r, r, r, indexing="ij"), -1).reshape(-1, 3)


def test_halo_plan_splits_phases_when_halo_exceeds_capacity():
    g, _ = P.build_from_coords(dense_cube(24))
    km = P.build_kernel_map(g, g, 1)
    plan = check_plan(km.fwd, 128, 128)  # 128 channels: ~288-slot capacity < a dense tile's ~400-row halo
    assert (plan.tensors["tile_level"] > 1).any()


CASES = [(32, 32), (64, 64), (128, 128), (64, 128), (128, 64), (32, 64), (128, 32)]


@pytest.fixture(scope="module")
def shell():
    c = sphere_shell_coords(48, band=1.5)
    g, _ = P.build_from_coords(c)
    og = O.build_from_coords(c)
    ins, outs = O.kernel_map(og, og, 1)
    return g, ins, outs, P.build_kernel_map(g, g, 1)


@pytest.mark.parametrize("cin,cout", CASES)
def test_halo_conv_matches_oracle_and_gather(shell, cin, cout):
    g, ins, outs, km = shell
    rng = np.random.default_rng(cin * 7 + cout)
    n = g.num_voxels
    x = rng.normal(size=(n, cin)).astype(np.float32)
    w = (rng.normal(size=(cout, cin, 3, 3, 3)) / np.sqrt(27 * cin)).astype(np.float32)
    gy = rng.normal(size=(n, cout)).astype(np.float32)
    xb = torch.from_numpy(x).cuda().to(torch.bfloat16)
    gyb = torch.from_numpy(gy).cuda().to(torch.bfloat16)
    wt = torch.from_numpy(w).cuda()
    ref_r = O.conv_igemm(bf16_round(x), bf16_round(w), ins, outs, n)
    y = gather_conv(xb, km.fwd, wt, out_dtype=torch.float32, impl="halo")
    assert rel(y, ref_r) < 2e-5
    yg = gather_conv(xb, km.fwd, wt, out_dtype=torch.float32, impl="gather")
    assert rel(y, yg.cpu().numpy()) < 2e-5
    y16 = gather_conv(xb, km.fwd, wt, impl="halo")
    ref = O.conv_igemm(x.astype(np.float64), w.astype(np.float64), ins, outs, n)
    assert y16.dtype == torch.bfloat16 and rel(y16, ref) < 1e-2
    gi_r, _ = O.conv_backward(ins, outs, bf16_round(gy), bf16_round(x), bf16_round(w))
    gi = gather_conv(gyb, km.bwd, wt, transpose=True, out_dtype=torch.float32, impl="halo")
    assert rel(gi, gi_r) < 2e-5


def test_halo_conv_phases_and_stride2():
    """Dense cube at 128 channels (multi-phase tiles) and a stride-2 map plus its transpose."""
    c = dense_cube(20)
    g, _ = P.build_from_coords(c)
    og = O.build_from_coords(c)
    rng = np.random.default_rng(5)
    for stride, K, N in ((1, 128, 128), (2, 64, 128), (2, 128, 64)):
        go, ogo = (g, og) if stride == 1 else (P.coarsen(g, 2), O.coarsen(og, 2))
        km = P.build_kernel_map(g, go, stride)
        ins, outs = O.kernel_map(og, ogo, stride)
        x = rng.normal(size=(g.num_voxels, K)).astype(np.float32)
        w = (rng.normal(size=(N, K, 3, 3, 3)) / np.sqrt(27 * K)).astype(np.float32)
        y = gather_conv(torch.from_numpy(x).cuda().to(torch.bfloat16), km.fwd, torch.from_numpy(w).cuda(),
                        out_dtype=torch.float32, impl="halo")
        assert rel(y, O.conv_igemm(bf16_round(x), bf16_round(w), ins, outs, go.num_voxels)) < 2e-5
        gy = rng.normal(size=(go.num_voxels, N)).astype(np.float32)
        gi = gather_conv(torch.from_numpy(gy).cuda().to(torch.bfloat16), km.bwd, torch.from_numpy(w).cuda(),
                         transpose=True, out_dtype=torch.float32, impl="halo")
        gi_r, _ = O.conv_backward(ins, outs, bf16_round(gy), bf16_round(x), bf16_round(w))
        assert rel(gi, gi_r) < 2e-5
    if stride == 1:
        pass


@pytest.mark.parametrize("cap", [256, 320])
@pytest.mark.parametrize("K,N", [(32, 32), (32, 64)])
def test_halo_offset_pairs_across_phases(K, N, cap):
    """K = 32 runs offset-pair stages (offsets 2v, 2v+1 as one 64-deep MMA K); a pair split by a phase
    boundary runs in both phases with the other half masked.  Plans at small capacities force 3-, 9- and
    27-phase tiles on a dense cube; fwd and dgrad must match the oracle."""
    from paper_2407_01781_b200.conv import HaloPlan
    c = dense_cube(20)
    g, _ = P.build_from_coords(c)
    og = O.build_from_coords(c)
    km = P.build_kernel_map(g, g, 1)
    ins, outs = O.kernel_map(og, og, 1)
    kcap = int(P._lib.lib().fvdb_halo_cap(K, N))
    for tab in (km.fwd, km.bwd):
        tab._plans[kcap] = HaloPlan(tab, cap)
    assert (km.fwd._plans[kcap].tensors["tile_level"] > 1).any()
    rng = np.random.default_rng(K + N + cap)
    n = g.num_voxels
    x = rng.normal(size=(n, K)).astype(np.float32)
    w = (rng.normal(size=(N, K, 3, 3, 3)) / np.sqrt(27 * K)).astype(np.float32)
    y = gather_conv(torch.from_numpy(x).cuda().to(torch.bfloat16), km.fwd, torch.from_numpy(w).cuda(),
                    out_dtype=torch.float32, impl="halo")
    assert rel(y, O.conv_igemm(bf16_round(x), bf16_round(w), ins, outs, n)) < 2e-5
    # dgrad: K input channels of the transposed conv = N
    w2 = (rng.normal(size=(K, N, 3, 3, 3)) / np.sqrt(27 * K)).astype(np.float32)
    gy = rng.normal(size=(n, K)).astype(np.float32)
    gi = gather_conv(torch.from_numpy(gy).cuda().to(torch.bfloat16), km.bwd, torch.from_numpy(w2).cuda(),
                     transpose=True, out_dtype=torch.float32, impl="halo")
    gi_r, _ = O.conv_backward(ins, outs, bf16_round(gy), bf16_round(np.zeros((n, N), np.float32)), bf16_round(w2))
    assert rel(gi, gi_r) < 2e-5


@pytest.mark.parametrize("K,N", [(64, 64), (32, 32), (32, 64), (64, 32)])
def test_dgrad_runs_the_forward_plan_reversed(K, N):
    """A same-grid stride-1 map's transposed table is its forward table with the offset rows reversed; the dgrad
    runs the forward plan with offsets_reversed = 1 (phases in reverse order, record offset 26 - d).  Small-capacity
    plans force multi-phase tiles."""
    from paper_2407_01781_b200.conv import HaloPlan
    c = dense_cube(20)
    g, _ = P.build_from_coords(c)
    og = O.build_from_coords(c)
    km = P.build_kernel_map(g, g, 1)
    ins, outs = O.kernel_map(og, og, 1)
    kcap = int(P._lib.lib().fvdb_halo_cap(N, K))
    km.fwd._plans[kcap] = HaloPlan(km.fwd, 256)
    assert (km.fwd._plans[kcap].tensors["tile_level"] > 1).any()
    plan = km.bwd.halo_plan(N, K)
    assert plan.c.offsets_reversed == 1 and plan.tensors is km.fwd._plans[kcap].tensors
    check_plan(km.bwd, N, K)
    rng = np.random.default_rng(K * 3 + N)
    n = g.num_voxels
    w = (rng.normal(size=(N, K, 3, 3, 3)) / np.sqrt(27 * K)).astype(np.float32)
    gy = rng.normal(size=(n, N)).astype(np.float32)
    gi = gather_conv(torch.from_numpy(gy).cuda().to(torch.bfloat16), km.bwd, torch.from_numpy(w).cuda(),
                     transpose=True, out_dtype=torch.float32, impl="halo")
    gi_r, _ = O.conv_backward(ins, outs, bf16_round(gy), bf16_round(np.zeros((n, K), np.float32)), bf16_round(w))
    assert rel(gi, gi_r) < 2e-5


def test_halo_conv_without_colours_and_deterministic(shell):
    """A KernelMap built from reference lists has no grids (no lane colours): same results."""
    g, ins, outs, km = shell
    km2 = P.KernelMap(ins, outs, g.num_voxels, g.num_voxels, 1)
    rng = np.random.default_rng(3)
    xb = torch.from_numpy(rng.normal(size=(g.num_voxels, 64)).astype(np.float32)).cuda().to(torch.bfloat16)
    w = torch.randn(64, 64, 3, 3, 3, device="cuda") / 40
    a = gather_conv(xb, km.fwd, w, out_dtype=torch.float32, impl="halo")
    b = gather_conv(xb, km2.fwd, w, out_dtype=torch.float32, impl="halo")
    assert rel(a, b.cpu().numpy()) < 1e-6
    assert torch.equal(a, gather_conv(xb, km.fwd, w, out_dtype=torch.float32, impl="halo"))


def test_halo_empty_and_tiny():
    g, _ = P.build_from_coords(np.array([[0, 0, 0]]))
    km = P.build_kernel_map(g, g, 1)
    x = torch.ones(1, 64, device="cuda", dtype=torch.bfloat16)
    w = torch.ones(64, 64, 3, 3, 3, device="cuda") / 64
    y = gather_conv(x, km.fwd, w, out_dtype=torch.float32, impl="halo")
    assert torch.allclose(y, torch.ones_like(y))


@pytest.mark.slow
def test_cfg2_full_size_halo_vs_torch_fp64():
    """BASELINE cfg2 (1,018,216 voxels, 64->64): the halo kernels the bench times, forward and dgrad, against
    a torch float64 per-offset reference of the same bf16-exact inputs (accumulation error only)."""
    g, _ = P.build_from_coords(sphere_shell_coords(470, band=1.5))
    km = P.build_kernel_map(g, g, 1)
    n = g.num_voxels
    gen = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(n, 64, device="cuda", generator=gen).to(torch.bfloat16)
    gy = torch.randn(n, 64, device="cuda", generator=gen).to(torch.bfloat16)
    w = torch.randn(64, 64, 3, 3, 3, device="cuda", generator=gen) / (27 * 64) ** 0.5
    y = gather_conv(x, km.fwd, w, out_dtype=torch.float32, impl="halo")
    gi = gather_conv(gy, km.bwd, w, transpose=True, out_dtype=torch.float32, impl="halo")
    wd = w.to(torch.bfloat16).double().reshape(64, 64, 27)
    xd, gyd, nbr = x.double(), gy.double(), km.nbr.long()
    ref_y = torch.zeros(n, 64, dtype=torch.float64, device="cuda")
    ref_gi = torch.zeros_like(ref_y)
    for d in range(27):
        m = nbr[d] >= 0
        o, i = torch.nonzero(m).squeeze(1), nbr[d][m]
        ref_y[o] += xd[i] @ wd[:, :, d].T
        ref_gi.index_add_(0, i, gyd[o] @ wd[:, :, d])
    for got, ref in ((y, ref_y), (gi, ref_gi)):
        assert float((got.double() - ref).abs().max() / ref.abs().max()) < 2e-5


@pytest.mark.slow
def test_cfg5_full_size_halo_adjoint_and_determinism():
    """BASELINE cfg5 (2048^3 shell, ~19.4M voxels, 32->32) at full size through size-independent
    properties: <conv(x), y> = <x, conv^T(y)> (forward and dgrad kernels are each other's adjoint) and
    bitwise run-to-run reproducibility."""
    g, _ = P.build_from_coords(sphere_shell_coords(2048, band=1.5))
    km = P.build_kernel_map(g, g, 1)
    n = g.num_voxels
    assert n > 19_000_000
    gen = torch.Generator(device="cuda").manual_seed(2)
    x = torch.randn(n, 32, device="cuda", generator=gen).to(torch.bfloat16)
    yv = torch.randn(n, 32, device="cuda", generator=gen).to(torch.bfloat16)
    w = torch.randn(32, 32, 3, 3, 3, device="cuda", generator=gen) / (27 * 32) ** 0.5
    cx = gather_conv(x, km.fwd, w, out_dtype=torch.float32, impl="halo")
    cty = gather_conv(yv, km.bwd, w, transpose=True, out_dtype=torch.float32, impl="halo")
    lhs = float((cx.double() * yv.double()).sum())
    rhs = float((x.double() * cty.double()).sum())
    scale = float((cx.double().abs() * yv.double().abs()).sum())
    assert abs(lhs - rhs) / scale < 1e-6
    assert torch.equal(cx, gather_conv(x, km.fwd, w, out_dtype=torch.float32, impl="halo"))
    # wgrad is the adjoint of the weight -> output map: <wgrad(x, y), W> = <conv(x; W), y>
    from paper_2407_01781_b200.conv import wgrad
    gw = wgrad(x, yv, km.fwd)
    wb = w.to(torch.bfloat16).double()
    lhs_w = float((gw.double() * wb).sum())
    scale_w = float((gw.double().abs() * wb.abs()).sum())
    assert abs(lhs_w - lhs) / scale_w < 1e-5


def test_variant_selects_dense_window_schedule():
    """variant="leaf"/"brick" (the reference's dense-window schedules, conv.py:200-261) run the halo kernel from
    the first call; "igemm" keeps the gather kernel for a fresh map; all compute the same operator."""
    r = np.arange(24)
    coords = np.stack(np.meshgrid(r, r, r, indexing="ij"), -1).reshape(-1, 3)
    g, _ = P.build_from_coords(coords)
    rng = np.random.default_rng(4)
    x = torch.from_numpy(rng.normal(size=(g.num_voxels, 64)).astype(np.float32)).cuda().to(torch.bfloat16)
    w = torch.from_numpy((rng.normal(size=(64, 64, 3, 3, 3)) / np.sqrt(27 * 64)).astype(np.float32))
    km = P.build_kernel_map(g, g, 1)
    y_igemm = P.conv(g, x, w, variant="igemm", kmap=km)
    assert not km.fwd.has_plan(64, 64)
    for v in ("leaf", "brick"):
        y = P.conv(g, x, w, variant=v, kmap=km)
        assert km.fwd.has_plan(64, 64)
        assert float((y.float() - y_igemm.float()).abs().max()) <= 2e-2 * float(y_igemm.float().abs().max())
    assert P.choose_variant(g, 64, 64) == "brick"  # 100% leaf occupancy
    y_auto = P.conv(g, x, w, variant="auto", kmap=km)
    assert torch.equal(y_auto, P.conv(g, x, w, variant="brick", kmap=km))


@pytest.mark.parametrize("case", ["shell", "cube_phases"])
def test_wgrad_on_halo_plan_matches_oracle(case, shell):
    """fvdb_conv_wgrad_halo (Cin = Cout = 32: xᵀ built in TMEM from the halo by ldmatrix.trans) against the oracle
    on bf16-rounded inputs and against the table kernel; multi-phase plans forced on a dense cube."""
    from paper_2407_01781_b200 import _lib
    from paper_2407_01781_b200.conv import C, HaloPlan
    if case == "shell":
        g, ins, outs, km = shell
    else:
        c = dense_cube(20)
        g, _ = P.build_from_coords(c)
        og = O.build_from_coords(c)
        km = P.build_kernel_map(g, g, 1)
        ins, outs = O.kernel_map(og, og, 1)
    rng = np.random.default_rng(17)
    n = g.num_voxels
    x = rng.normal(size=(n, 32)).astype(np.float32)
    gy = rng.normal(size=(n, 32)).astype(np.float32)
    kcap = int(_lib.lib().fvdb_halo_cap(32, 32))
    plan = HaloPlan(km.fwd, kcap if case == "shell" else 256)
    if case != "shell":
        assert (plan.tensors["tile_level"] > 1).any()
    xb = torch.from_numpy(x).cuda().to(torch.bfloat16)
    gyb = torch.from_numpy(gy).cuda().to(torch.bfloat16)
    L = _lib.lib()
    gw = torch.empty((32, 32, 3, 3, 3), dtype=torch.float32, device="cuda")
    wsb = L.fvdb_wgrad_halo_workspace_bytes(n)
    ws = _lib.workspace(wsb, "cuda")
    _lib.check(L.fvdb_conv_wgrad_halo(xb.data_ptr(), n, 32, gyb.data_ptr(), 32, C.byref(plan.c), n, gw.data_ptr(),
                                      ws.data_ptr(), wsb, _lib.stream_ptr()), "wgrad_halo")
    _, gw_r = O.conv_backward(ins, outs, bf16_round(gy), bf16_round(x), np.zeros((32, 32, 3, 3, 3)))
    assert rel(gw, gw_r) < 2e-5
    from paper_2407_01781_b200.conv import wgrad
    import os
    os.environ["FVDB_WG_HALO"] = "0"
    try:
        gw_t = wgrad(xb, gyb, km.fwd)  # the table kernel
    finally:
        del os.environ["FVDB_WG_HALO"]
    assert rel(gw, gw_t.cpu().numpy()) < 2e-5


def test_halo_conv_repeated_runs_identical():
    """Stress for races between the halo kernel's warps: 200 forwards on the cfg2 shell (64x64: two halo loader
    warps, multi-phase tiles such as tile 2, the plan's first, which is also CTA 2's first tile), each compared
    bitwise with the first and within 2e-5 with the gather kernel.  The second loader warp once read a row-id
    buffer the first had already refilled: 2 of 300 runs wrong (tools/halo_stress.py)."""
    g, _ = P.build_from_coords(sphere_shell_coords(470, band=1.5))
    km = P.build_kernel_map(g, g, 1)
    gen = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(g.num_voxels, 64, device="cuda", generator=gen).to(torch.bfloat16)
    w = torch.randn(64, 64, 3, 3, 3, device="cuda", generator=gen) / (27 * 64) ** 0.5
    ref = gather_conv(x, km.fwd, w, out_dtype=torch.float32, impl="gather")
    first = gather_conv(x, km.fwd, w, out_dtype=torch.float32, impl="halo")
    assert int(km.fwd.halo_plan(64, 64).tensors["tile_level"][2]) > 1  # the case that exposed the race
    assert rel(first, ref.cpu().numpy()) < 2e-5
    bad = 0
    for _ in range(200):
        y = gather_conv(x, km.fwd, w, out_dtype=torch.float32, impl="halo")
        bad += int(not torch.equal(y, first))
    assert bad == 0
