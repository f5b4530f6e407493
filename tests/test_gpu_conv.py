"""GPU parity: sparse conv forward / dgrad / wgrad / transposed / module vs the oracle.

Tolerances (BASELINE.json north star): fp32 path rel 1e-5, f64 path rel 1e-10 (reference
test_conv.py:137-146), bf16 tensor-core path rel 1e-2 against the reference fp32 output.
rel = max|Δ| / max|ref|.  The bf16 kernels are additionally checked against the oracle on
the bf16-rounded inputs (isolates accumulation error; fp32 TMEM accumulation → ≤ 2e-5).
"""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.conv import gather_conv, wgrad
from paper_2407_01781_b200.workloads import sphere_shell_coords
from conftest import CONV_CASES

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = a.detach().double().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def bf16_round(a):
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).float().numpy().astype(np.float64)


def grids(golden_grids, name, stride):
    c = golden_grids[f"{name}/coords"]
    g, _ = P.build_from_coords(c)
    og = O.build_from_coords(c)
    if stride == 1:
        return g, g, og, og
    return g, P.coarsen(g, 2), og, O.coarsen(og, 2)


@pytest.mark.parametrize("name", CONV_CASES)
@pytest.mark.parametrize("stride", [1, 2])
def test_simt_forward_backward_match_reference(golden_grids, golden_convs, name, stride):
    g, go_grid, _, _ = grids(golden_grids, name, stride)
    km = P.build_kernel_map(g, go_grid, stride)
    k = f"{name}/s{stride}"
    f64, w64, go64 = golden_convs[f"{k}/features"], golden_convs[f"{k}/weights"], golden_convs[f"{k}/grad_out"]
    out = P.conv(g, f64, w64, grid_out=go_grid, stride=stride, kmap=km)
    assert out.dtype == torch.float64
    assert rel(out, golden_convs[f"{k}/out_f64"]) < 1e-10
    gi, gw = P.conv_backward(km, go64, f64, w64)
    assert rel(gi, golden_convs[f"{k}/grad_in_f64"]) < 1e-10
    assert rel(gw, golden_convs[f"{k}/grad_w_f64"]) < 1e-10
    f32, w32, go32 = (a.astype(np.float32) for a in (f64, w64, go64))
    out = P.conv(g, f32, w32, grid_out=go_grid, stride=stride, kmap=km)
    assert out.dtype == torch.float32
    assert rel(out, golden_convs[f"{k}/out_f32"]) < 1e-5
    assert rel(out, golden_convs[f"{k}/out_f64"]) < 1e-5
    gi, gw = P.conv_backward(km, go32, f32, w32)
    assert rel(gi, golden_convs[f"{k}/grad_in_f32"]) < 1e-5
    assert rel(gw, golden_convs[f"{k}/grad_w_f32"]) < 1e-5


def test_reference_fixture_conv(golden_fixtures):
    fx = golden_fixtures
    g, _ = P.build_from_points(fx["points"], P.VoxelTransform(fx["voxel_size"], fx["origin"]))
    out = P.conv(g, fx["conv_features"], fx["conv_weights"], variant="igemm")
    assert rel(out, fx["conv_expected"]) < 1e-12


@pytest.mark.parametrize("variant", ["igemm", "leaf", "brick", "lggs", "auto"])
def test_variants_identity_and_all_ones(variant):
    rng = np.random.default_rng(2)
    g, _ = P.build_from_coords(rng.integers(-15, 15, size=(400, 3)))
    f = rng.normal(size=(g.num_voxels, 5))
    out = P.conv(g, f, P.ConvKernel.identity(5), variant=variant)
    assert np.allclose(out.cpu().numpy(), f)
    blk = np.stack(np.meshgrid(*[np.arange(3)] * 3, indexing="ij"), -1).reshape(-1, 3)
    g, _ = P.build_from_coords(blk)
    out = P.conv(g, np.ones((27, 1)), np.ones((1, 1, 3, 3, 3)), variant=variant).cpu().numpy()
    assert out[g.coord_to_index(1, 1, 1) - 1, 0] == 27 and out[g.coord_to_index(0, 0, 0) - 1, 0] == 8


def test_lggs_stats_and_errors():
    rng = np.random.default_rng(7)
    g, _ = P.build_from_coords(rng.integers(-25, 25, size=(3000, 3)))
    stats = {}
    P.conv(g, rng.normal(size=(g.num_voxels, 4)).astype(np.float32),
           rng.normal(size=(4, 4, 3, 3, 3)).astype(np.float32), variant="lggs", stats=stats)
    assert 0 < stats["lggs_pad_rows_max"] <= 15
    assert stats["lggs_blocks"] == (g.num_voxels + 63) // 64
    g1, _ = P.build_from_coords([(0, 0, 0)])
    with pytest.raises(ValueError, match="variant"):
        P.conv(g1, np.ones((1, 1)), np.ones((1, 1, 3, 3, 3)), variant="wavelet")
    with pytest.raises(ValueError, match="features"):
        P.conv(g1, np.ones((4, 1)), np.ones((1, 1, 3, 3, 3)))
    with pytest.raises(ValueError, match="stride"):
        P.conv(g1, np.ones((1, 1)), np.ones((1, 1, 3, 3, 3)), variant="lggs", stride=2)
    km = P.build_kernel_map(g1, g1, 1)
    with pytest.raises(ValueError, match="grad_out"):
        P.conv_backward(km, np.zeros((2, 2)), np.zeros((1, 3)), np.zeros((2, 3, 3, 3, 3)))


def test_linearity_and_batch_bitwise():
    rng = np.random.default_rng(5)
    g, _ = P.build_from_coords(rng.integers(-10, 10, size=(250, 3)))
    x, y = rng.normal(size=(g.num_voxels, 4)), rng.normal(size=(g.num_voxels, 4))
    w = rng.normal(size=(3, 4, 3, 3, 3))
    lhs = P.conv(g, 1.7 * x - 0.4 * y, w).cpu().numpy()
    rhs = 1.7 * P.conv(g, x, w).cpu().numpy() - 0.4 * P.conv(g, y, w).cpu().numpy()
    assert np.allclose(lhs, rhs, atol=1e-12)
    rng = np.random.default_rng(12)
    gl = [P.build_from_coords(rng.integers(-s, s, size=(n, 3)))[0] for s, n in ((8, 120), (14, 300))]
    gb = P.grid_batch(gl)
    for dt in (np.float64, np.float32):
        feats = gb.jagged(rng.normal(size=(gb.total_voxels, 4)).astype(dt))
        out = P.conv_batch(gb, feats, rng.normal(size=(3, 4, 3, 3, 3)).astype(dt))
        w = rng.normal(size=(3, 4, 3, 3, 3)).astype(dt)
        out = P.conv_batch(gb, feats, w)
        for b, gg in enumerate(gl):
            assert torch.equal(out.element(b), P.conv(gg, feats.element(b), w))


def test_backward_finite_differences_f64():
    rng = np.random.default_rng(0)
    g, _ = P.build_from_coords(rng.integers(-6, 6, size=(120, 3)))
    n = g.num_voxels
    f, w, go = rng.normal(size=(n, 3)), rng.normal(size=(2, 3, 3, 3, 3)), rng.normal(size=(n, 2))
    km = P.build_kernel_map(g, g, 1)
    gi, gw = (t.cpu().numpy() for t in P.conv_backward(km, go, f, w))

    def loss(ff, ww):
        return float(np.sum(go * P.conv(g, ff, ww, kmap=km).cpu().numpy()))

    h = 1e-6
    for _ in range(8):
        r, c = rng.integers(0, n), rng.integers(0, 3)
        fp, fm = f.copy(), f.copy()
        fp[r, c] += h
        fm[r, c] -= h
        fd = (loss(fp, w) - loss(fm, w)) / (2 * h)
        assert abs(fd - gi[r, c]) <= 1e-6 * max(1.0, abs(fd))
    for _ in range(8):
        co, ci = rng.integers(0, 2), rng.integers(0, 3)
        a, b, c3 = rng.integers(0, 3, size=3)
        wp, wm = w.copy(), w.copy()
        wp[co, ci, a, b, c3] += h
        wm[co, ci, a, b, c3] -= h
        fd = (loss(f, wp) - loss(f, wm)) / (2 * h)
        assert abs(fd - gw[co, ci, a, b, c3]) <= 1e-6 * max(1.0, abs(fd))


# ---------------------------------------------------------------- tensor cores

TC_SHAPES = [(32, 32), (64, 64), (128, 128), (32, 64), (64, 32), (64, 128), (128, 64), (128, 32)]


@pytest.fixture(scope="module")
def shell():
    c = sphere_shell_coords(48, band=1.5)
    g, _ = P.build_from_coords(c)
    og = O.build_from_coords(c)
    ins, outs = O.kernel_map(og, og, 1)
    return g, og, ins, outs, P.build_kernel_map(g, g, 1)


@pytest.mark.parametrize("cin,cout", TC_SHAPES)
def test_tc_forward_dgrad_wgrad(shell, cin, cout):
    g, og, ins, outs, km = shell
    rng = np.random.default_rng(cin * 1000 + cout)
    n = g.num_voxels
    x = rng.normal(size=(n, cin)).astype(np.float32)
    w = (rng.normal(size=(cout, cin, 3, 3, 3)) / np.sqrt(27 * cin)).astype(np.float32)
    gy = rng.normal(size=(n, cout)).astype(np.float32)
    xr, wr, gyr = bf16_round(x), bf16_round(w), bf16_round(gy)
    xb = torch.from_numpy(x).cuda().to(torch.bfloat16)
    gyb = torch.from_numpy(gy).cuda().to(torch.bfloat16)
    wt = torch.from_numpy(w).cuda()
    # forward
    ref_r = O.conv_igemm(xr, wr, ins, outs, n)
    ref = O.conv_igemm(x.astype(np.float64), w.astype(np.float64), ins, outs, n)
    y32 = gather_conv(xb, km.fwd, wt, out_dtype=torch.float32)
    assert rel(y32, ref_r) < 2e-5
    y16 = gather_conv(xb, km.fwd, wt)
    assert y16.dtype == torch.bfloat16
    assert rel(y16, ref) < 1e-2
    # dgrad
    gi_r, gw_r = O.conv_backward(ins, outs, gyr, xr, wr)
    gi32 = gather_conv(gyb, km.bwd, wt, transpose=True, out_dtype=torch.float32)
    assert rel(gi32, gi_r) < 2e-5
    gi_ref, gw_ref = O.conv_backward(ins, outs, gy.astype(np.float64), x.astype(np.float64), w.astype(np.float64))
    assert rel(gather_conv(gyb, km.bwd, wt, transpose=True), gi_ref) < 1e-2
    # wgrad
    gw = wgrad(xb, gyb, km.fwd)
    assert gw.dtype == torch.float32 and tuple(gw.shape) == (cout, cin, 3, 3, 3)
    assert rel(gw, gw_r) < 2e-5
    assert rel(gw, gw_ref) < 1e-2


def test_tc_deterministic(shell):
    g, og, ins, outs, km = shell
    rng = np.random.default_rng(1)
    xb = torch.from_numpy(rng.normal(size=(g.num_voxels, 64)).astype(np.float32)).cuda().to(torch.bfloat16)
    gyb = torch.from_numpy(rng.normal(size=(g.num_voxels, 64)).astype(np.float32)).cuda().to(torch.bfloat16)
    w = torch.randn(64, 64, 3, 3, 3, device="cuda")
    a = gather_conv(xb, km.fwd, w, out_dtype=torch.float32)
    b = gather_conv(xb, km.fwd, w, out_dtype=torch.float32)
    assert torch.equal(a, b)
    assert torch.equal(wgrad(xb, gyb, km.fwd), wgrad(xb, gyb, km.fwd))


def test_tc_unaligned_channels_pad(shell):
    g, og, ins, outs, km = shell
    rng = np.random.default_rng(9)
    x = rng.normal(size=(g.num_voxels, 20)).astype(np.float32)
    w = rng.normal(size=(40, 20, 3, 3, 3)).astype(np.float32) / 20
    y = P.conv(g, torch.from_numpy(x).cuda().to(torch.bfloat16), w, kmap=km)
    ref = O.conv_igemm(x.astype(np.float64), w.astype(np.float64), ins, outs, g.num_voxels)
    assert rel(y, ref) < 1e-2


def test_tc_stride2_and_transposed():
    rng = np.random.default_rng(3)
    c = sphere_shell_coords(40, band=1.5)
    g, _ = P.build_from_coords(c)
    g2 = P.coarsen(g, 2)
    og = O.build_from_coords(c)
    og2 = O.coarsen(og, 2)
    ins, outs = O.kernel_map(og, og2, 2)
    km = P.build_kernel_map(g, g2, 2)
    x = rng.normal(size=(g.num_voxels, 64)).astype(np.float32)
    w = (rng.normal(size=(128, 64, 3, 3, 3)) / np.sqrt(27 * 64)).astype(np.float32)
    xb = torch.from_numpy(x).cuda().to(torch.bfloat16)
    y = P.conv(g, xb, w, grid_out=g2, stride=2, kmap=km)
    assert rel(y, O.conv_igemm(x.astype(np.float64), w.astype(np.float64), ins, outs, g2.num_voxels)) < 1e-2
    # transposed 128 -> 64 with W [C_coarse=128, C_fine=64]
    wt = (rng.normal(size=(128, 64, 3, 3, 3)) / np.sqrt(27 * 128)).astype(np.float32)
    z = rng.normal(size=(g2.num_voxels, 128)).astype(np.float32)
    yt = P.conv_transpose(km, torch.from_numpy(z).cuda().to(torch.bfloat16), wt, out_dtype=torch.float32)
    ref = O.conv_transpose(ins, outs, bf16_round(z), bf16_round(wt), g.num_voxels)
    assert rel(yt, ref) < 2e-5
    # f64 transposed = conv_backward(...)[0] and adjoint identity
    z64 = rng.normal(size=(g2.num_voxels, 7))
    w64 = rng.normal(size=(7, 5, 3, 3, 3))
    x64 = rng.normal(size=(g.num_voxels, 5))
    yt64 = P.conv_transpose(km, z64, w64).cpu().numpy()
    assert rel(yt64, O.conv_transpose(ins, outs, z64, w64, g.num_voxels)) < 1e-12
    lhs = np.sum(P.conv(g, x64, w64, grid_out=g2, stride=2, kmap=km).cpu().numpy() * z64)
    assert abs(lhs - np.sum(x64 * yt64)) <= 1e-10 * abs(lhs)


@pytest.mark.parametrize("mode", ["s1", "s2", "transposed"])
@pytest.mark.parametrize("cdt", [torch.bfloat16, torch.float32])
def test_sparseconv3d_module_autograd(mode, cdt):
    rng = np.random.default_rng(11)
    grids_c = [sphere_shell_coords(24, band=1.5), rng.integers(-12, 12, size=(600, 3))]
    fine = P.GridBatch([P.build_from_coords(c)[0] for c in grids_c])
    ofine = [O.build_from_coords(c) for c in grids_c]
    cin, cout = 64, 32
    if mode == "transposed":
        coarse = P.GridBatch([P.coarsen(g, 2) for g in fine.grids])
        m = P.SparseConv3d(cin, cout, stride=2, transposed=True, compute_dtype=cdt).cuda()
        src_batch, n_src = coarse, coarse.total_voxels
    else:
        m = P.SparseConv3d(cin, cout, stride=1 if mode == "s1" else 2, compute_dtype=cdt).cuda()
        src_batch, n_src = fine, fine.total_voxels
    x = torch.randn(n_src, cin, device="cuda", requires_grad=True)
    if mode == "transposed":
        out_grid, y = m(src_batch, src_batch.jagged(x), out_grid=fine)
    else:
        out_grid, y = m(src_batch, src_batch.jagged(x))
    gy = torch.randn_like(y.jdata.float())
    (y.jdata.float() * gy).sum().backward()
    w = m.weight.detach().cpu().double().numpy()
    # oracle per element
    xs = x.detach().cpu().double().numpy()
    gys = gy.cpu().double().numpy()
    tol = 1e-2 if cdt == torch.bfloat16 else 1e-5
    ys, gxs, gws = [], [], np.zeros_like(w)
    for b, og in enumerate(ofine):
        if mode == "s1":
            ins, outs = O.kernel_map(og, og, 1)
            xi = xs[src_batch.voxel_slice(b)]
            ys.append(O.conv_igemm(xi, w, ins, outs, og.num_voxels))
            gi, gw = O.conv_backward(ins, outs, gys[out_grid.voxel_slice(b)], xi, w)
        elif mode == "s2":
            og2 = O.coarsen(og, 2)
            ins, outs = O.kernel_map(og, og2, 2)
            xi = xs[src_batch.voxel_slice(b)]
            ys.append(O.conv_igemm(xi, w, ins, outs, og2.num_voxels))
            gi, gw = O.conv_backward(ins, outs, gys[out_grid.voxel_slice(b)], xi, w)
        else:
            og2 = O.coarsen(og, 2)
            ins, outs = O.kernel_map(og, og2, 2)
            zi = xs[src_batch.voxel_slice(b)]
            ys.append(O.conv_transpose(ins, outs, zi, w, og.num_voxels))
            gyi = gys[out_grid.voxel_slice(b)]
            gi = O.conv_igemm(gyi, w, ins, outs, og2.num_voxels)      # dgrad of transposed = s2 conv
            gw = O.conv_backward(ins, outs, zi, gyi, w)[1]             # roles swapped
        gxs.append(gi)
        gws += gw
    assert rel(y.jdata, np.concatenate(ys)) < tol
    assert rel(x.grad, np.concatenate(gxs)) < tol
    assert rel(m.weight.grad, gws) < tol


@pytest.mark.slow
def test_cfg2_full_size_tc_vs_torch_fp64():
    """1M-voxel 64->64 layer: forward / dgrad / wgrad vs a torch float64 per-offset reference."""
    c = sphere_shell_coords(470, band=1.5)
    g, _ = P.build_from_coords(c)
    km = P.build_kernel_map(g, g, 1)
    n = g.num_voxels
    gen = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(n, 64, device="cuda", generator=gen).to(torch.bfloat16)
    gy = torch.randn(n, 64, device="cuda", generator=gen).to(torch.bfloat16)
    w = torch.randn(64, 64, 3, 3, 3, device="cuda", generator=gen) / (27 * 64) ** 0.5
    wr = w.to(torch.bfloat16).double()
    xd, gyd = x.double(), gy.double()
    nbr = km.nbr.long()
    y = gather_conv(x, km.fwd, w, out_dtype=torch.float32)
    gi = gather_conv(gy, km.bwd, w, transpose=True, out_dtype=torch.float32)
    gw = wgrad(x, gy, km.fwd)
    ref_y = torch.zeros(n, 64, dtype=torch.float64, device="cuda")
    ref_gi = torch.zeros_like(ref_y)
    ref_gw = torch.zeros(64, 64, 27, dtype=torch.float64, device="cuda")
    wd = wr.reshape(64, 64, 27)
    for d in range(27):
        m = nbr[d] >= 0
        o = torch.nonzero(m).squeeze(1)
        i = nbr[d][m]
        ref_y[o] += xd[i] @ wd[:, :, d].T
        ref_gi.index_add_(0, i, gyd[o] @ wd[:, :, d])
        ref_gw[:, :, d] = gyd[o].T @ xd[i]
    def r(a, b):
        return float((a.double() - b).abs().max() / b.abs().max())
    assert r(y, ref_y) < 2e-5
    assert r(gi, ref_gi) < 2e-5
    assert r(gw.reshape(64, 64, 27), ref_gw) < 2e-5


@pytest.mark.parametrize("cin,cout", [(64, 64), (40, 48), (8, 8), (32, 24)])
def test_simt_tiled_shapes_match_oracle(shell, cin, cout):
    """The tiled fp32/f64 kernel (K, N multiples of 8, N <= 64): several K chunks, a zero-padded last
    chunk (K = 40), both column tiles (N <= 32, N <= 64); forward and dgrad against the oracle."""
    g, _, ins, outs, km = shell
    rng = np.random.default_rng(cin * 13 + cout)
    n = g.num_voxels
    x = rng.normal(size=(n, cin))
    w = rng.normal(size=(cout, cin, 3, 3, 3)) / np.sqrt(27 * cin)
    gy = rng.normal(size=(n, cout))
    ref = O.conv_igemm(x, w, ins, outs, n)
    gi_ref, _ = O.conv_backward(ins, outs, gy, x, w)
    for dt, tol in ((torch.float64, 1e-10), (torch.float32, 1e-5)):
        xt, wt, gyt = (torch.from_numpy(a).cuda().to(dt) for a in (x, w, gy))
        assert rel(gather_conv(xt, km.fwd, wt), ref) < tol
        assert rel(gather_conv(gyt, km.bwd, wt, transpose=True), gi_ref) < tol


def test_wide_channels_blocked(shell):
    """Channel counts beyond the kernels' widths (the reference takes any): bf16 192 -> 256 through K / N
    blocks (fwd, dgrad, wgrad) and fp32 / f64 with N = 300 through column blocks, against the oracle."""
    g, _, ins, outs, km = shell
    n = g.num_voxels
    rng = np.random.default_rng(77)
    cin, cout = 192, 256
    x = rng.normal(size=(n, cin)).astype(np.float32)
    w = (rng.normal(size=(cout, cin, 3, 3, 3)) / np.sqrt(27 * cin)).astype(np.float32)
    gy = rng.normal(size=(n, cout)).astype(np.float32)
    xb, gyb = (torch.from_numpy(a).cuda().to(torch.bfloat16) for a in (x, gy))
    wt = torch.from_numpy(w).cuda()
    y = gather_conv(xb, km.fwd, wt, out_dtype=torch.float32)
    assert y.shape == (n, cout) and rel(y, O.conv_igemm(bf16_round(x), bf16_round(w), ins, outs, n)) < 2e-5
    gi_r, gw_r = O.conv_backward(ins, outs, bf16_round(gy), bf16_round(x), bf16_round(w))
    gi = gather_conv(gyb, km.bwd, wt, transpose=True, out_dtype=torch.float32)
    assert gi.shape == (n, cin) and rel(gi, gi_r) < 2e-5
    gw = wgrad(xb, gyb, km.fwd)
    assert gw.shape == (cout, cin, 3, 3, 3) and rel(gw, gw_r) < 2e-5
    x2 = rng.normal(size=(n, 20))
    w2 = rng.normal(size=(300, 20, 3, 3, 3)) / np.sqrt(27 * 20)
    ref2 = O.conv_igemm(x2, w2, ins, outs, n)
    for dt, tol in ((torch.float64, 1e-10), (torch.float32, 1e-5)):
        y2 = gather_conv(torch.from_numpy(x2).cuda().to(dt), km.fwd, torch.from_numpy(w2).cuda().to(dt))
        assert y2.shape == (n, 300) and rel(y2, ref2) < tol


@pytest.mark.parametrize("n,off", [(0, 0), (7, 0), (1 << 16, 0), ((1 << 16) + 5, 0), (1003, 1), (4096, 3)])
def test_f32_to_bf16_matches_torch(n, off):
    """fvdb_f32_to_bf16 (vectorised for 16-B aligned buffers, scalar otherwise) rounds to nearest even,
    bit-identical to torch's cast, including the unaligned and tail paths."""
    from paper_2407_01781_b200.nn import _to_compute
    src = (torch.randn(n + off, device="cuda") * 1e3)[off:]
    src[: min(n, 4)] = torch.tensor([float("inf"), float("-inf"), float("nan"), 3.0e38], device="cuda")[: min(n, 4)]
    got = _to_compute(src, torch.bfloat16)
    ref = src.to(torch.bfloat16)
    assert got.dtype == torch.bfloat16 and got.shape == ref.shape
    assert torch.equal(got.view(torch.int16), ref.view(torch.int16))


def test_module_input_grad_dtype():
    """SparseConv3d (bf16 compute): y in bf16, the fp32 input's gradient written in fp32 by the kernel."""
    g, _ = P.build_from_coords(sphere_shell_coords(24, band=1.5))
    gb = P.GridBatch([g])
    m = P.SparseConv3d(64, 64).cuda()
    x = torch.randn(g.num_voxels, 64, device="cuda", requires_grad=True)
    _, y = m(gb, gb.jagged(x))
    assert y.jdata.dtype == torch.bfloat16
    y.jdata.float().sum().backward()
    assert x.grad.dtype == torch.float32 and torch.isfinite(x.grad).all()


@pytest.mark.parametrize("dtype,tol", [(np.float32, 1e-5), (np.float64, 1e-10)])
@pytest.mark.parametrize("which", ["s1", "s2T"])
def test_exact_offset_skipping(monkeypatch, dtype, tol, which):
    """The exact-precision gather kernel with tile masks / over the signature-sorted table skips only
    zero-filled rows: bitwise equal to walking all 27 offsets, and within the exact-path tolerance of the
    oracle (conv.py:180-191; transposed form conv.py:339-368)."""
    c = sphere_shell_coords(30, band=1.5)
    g, _ = P.build_from_coords(c)
    og = O.build_from_coords(c)
    if which == "s1":
        km, (ins, outs), n_in, n_out = P.build_kernel_map(g, g, 1), O.kernel_map(og, og, 1), g.num_voxels, g.num_voxels
    else:
        gc, ogc = P.coarsen(g, 2), O.coarsen(og, 2)
        km, (ins, outs) = P.build_kernel_map(g, gc, 2), O.kernel_map(og, ogc, 2)
        n_in, n_out = gc.num_voxels, g.num_voxels
    rng = np.random.default_rng(11)
    x = rng.normal(size=(n_in, 32)).astype(dtype)
    w = (rng.normal(size=(32, 32, 3, 3, 3)) / np.sqrt(27 * 32)).astype(dtype)
    xt, wt = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    res = {}
    for mode in ("none", "masks", "sort"):
        monkeypatch.setenv("FVDB_EXACT_SKIP", mode)
        if which == "s1":
            res[mode] = gather_conv(xt, km.fwd, wt)
        else:
            res[mode] = gather_conv(xt, km.bwd, wt, transpose=True)
    assert torch.equal(res["none"], res["masks"]) and torch.equal(res["none"], res["sort"])
    if which == "s1":
        ref = O.conv_igemm(x.astype(np.float64), w.astype(np.float64), ins, outs, n_out)
    else:
        ref = O.conv_transpose(ins, outs, x.astype(np.float64), w.astype(np.float64), n_out)
    assert rel(res["sort"], ref) < tol
