"""GPU: weight gradient over per-offset pair lists (fvdb_kmap_pair_lists, fvdb_conv_wgrad_pairs_tc in
csrc/wgrad_pairs.cu) against the oracle's per-offset form gw[:,:,d] = go[outs[d]]ᵀ · x[ins[d]]
(conv.py:358-366), on bf16-rounded inputs with fp32 accumulation (rel <= 2e-5).
"""
import sys

import numpy as np
import pytest
import torch

import oracle as O
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.conv import wgrad, wgrad_pairs_enabled
from paper_2407_01781_b200.workloads import sphere_shell_coords

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = a.detach().double().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def bf16_round(a):
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).float().numpy().astype(np.float64)


@pytest.fixture(scope="module")
def maps():
    c = sphere_shell_coords(40, band=1.5)
    g, _ = P.build_from_coords(c)
    og = O.build_from_coords(c)
    gc, ogc = P.coarsen(g, 2), O.coarsen(og, 2)
    return {"s1": (g, g, P.build_kernel_map(g, g, 1), O.kernel_map(og, og, 1)),
            "s2": (g, gc, P.build_kernel_map(g, gc, 2), O.kernel_map(og, ogc, 2))}


@pytest.mark.parametrize("which", ["s1", "s2"])
def test_pair_lists_exact(maps, which):
    _, _, km, _ = maps[which]
    tab = km.fwd
    tab._pairs = None
    pin, pout, seg, total = tab.pair_lists()
    v = tab.view.cpu().numpy()
    seg = seg.cpu().numpy()
    assert seg[0] == 0 and seg[27] == total and (np.diff(seg) % 128 == 0).all()
    pin, pout = pin.cpu().numpy(), pout.cpu().numpy()
    for d in range(27):
        o = np.nonzero(v[d] >= 0)[0]
        a, b = seg[d], seg[d + 1]
        assert b - a == (len(o) + 127) // 128 * 128
        assert np.array_equal(pout[a:a + len(o)], o) and np.array_equal(pin[a:a + len(o)], v[d, o])
        assert (pout[a + len(o):b] == -1).all() and (pin[a + len(o):b] == -1).all()
    tp = tab.pair_tile_pos().cpu().numpy().reshape(27, -1)
    tiles = (tab.n + 127) // 128
    assert tp.shape == (27, tiles + 1)
    for d in range(27):
        o = np.nonzero(v[d] >= 0)[0]
        want = seg[d] + np.searchsorted(o, np.arange(tiles + 1) * 128)
        assert np.array_equal(tp[d], want)


SHAPES = [(128, 128), (64, 128), (128, 64), (32, 128), (128, 32)]


@pytest.mark.parametrize("sched", ["tiles", "linear"])
@pytest.mark.parametrize("which", ["s1", "s2"])
@pytest.mark.parametrize("cin,cout", SHAPES)
def test_wgrad_pairs_vs_oracle(maps, monkeypatch, which, cin, cout, sched):
    """Both schedules: linear shares of the offset-major lists (default) and offset groups x tile ranges."""
    monkeypatch.setattr(sys.modules["paper_2407_01781_b200.conv"], "_WG_PAIRS_SCHED", sched)
    g, go_grid, km, (ins, outs) = maps[which]
    rng = np.random.default_rng(cin + 7 * cout + (which == "s2"))
    x = rng.normal(size=(g.num_voxels, cin)).astype(np.float32)
    gy = rng.normal(size=(go_grid.num_voxels, cout)).astype(np.float32)
    w0 = np.zeros((cout, cin, 3, 3, 3))
    _, gw_r = O.conv_backward(ins, outs, bf16_round(gy), bf16_round(x), w0)
    xb = torch.from_numpy(x).cuda().to(torch.bfloat16)
    gyb = torch.from_numpy(gy).cuda().to(torch.bfloat16)
    monkeypatch.setenv("FVDB_WG_PAIRS", "force")
    assert wgrad_pairs_enabled(km.fwd, cin, cout)
    gw = wgrad(xb, gyb, km.fwd)
    assert gw.dtype == torch.float32 and tuple(gw.shape) == (cout, cin, 3, 3, 3)
    assert rel(gw, gw_r) < 2e-5
    assert torch.equal(gw, wgrad(xb, gyb, km.fwd))  # fixed reduction order
    monkeypatch.setenv("FVDB_WG_PAIRS", "0")
    assert rel(wgrad(xb, gyb, km.fwd), gw_r) < 2e-5


@pytest.mark.parametrize("sched", ["tiles", "linear"])
def test_wgrad_pairs_empty_offsets_and_tables(monkeypatch, sched):
    """Offsets without pairs get zero gradient; an empty table gives all zeros.  With one tile the
    tile-ordered schedule leaves most CTAs of the dense group with empty tile ranges (zero partials)."""
    monkeypatch.setattr(sys.modules["paper_2407_01781_b200.conv"], "_WG_PAIRS_SCHED", sched)
    monkeypatch.setenv("FVDB_WG_PAIRS", "force")
    g, _ = P.build_from_coords(np.array([[0, 0, 0], [0, 0, 1], [9, 9, 9]]))
    km = P.build_kernel_map(g, g, 1)
    x = torch.randn(3, 128, device="cuda").to(torch.bfloat16)
    gy = torch.randn(3, 64, device="cuda").to(torch.bfloat16)
    gw = wgrad(x, gy, km.fwd)
    og = O.build_from_coords(np.array([[0, 0, 0], [0, 0, 1], [9, 9, 9]]))
    ins, outs = O.kernel_map(og, og, 1)
    _, gw_r = O.conv_backward(ins, outs, gy.float().cpu().numpy().astype(np.float64),
                              x.float().cpu().numpy().astype(np.float64), np.zeros((64, 128, 3, 3, 3)))
    assert rel(gw, gw_r) < 2e-5
    assert int((gw.abs().sum((0, 1)) > 0).sum()) == 3  # centre and the two z-neighbour offsets
    ge = P.build_from_coords(np.zeros((0, 3), np.int64))[0]
    kme = P.build_kernel_map(ge, ge, 1)
    gwe = wgrad(torch.zeros(0, 128, device="cuda", dtype=torch.bfloat16),
                torch.zeros(0, 128, device="cuda", dtype=torch.bfloat16), kme.fwd)
    assert gwe.shape == (128, 128, 3, 3, 3) and not gwe.any()


def test_policy(maps, monkeypatch):
    from paper_2407_01781_b200.conv import NbrTable
    monkeypatch.delenv("FVDB_WG_PAIRS", raising=False)
    _, _, km1, _ = maps["s1"]
    assert km1.fwd.density() > 11 and not wgrad_pairs_enabled(km1.fwd, 64, 128)  # dense: table kernel
    sparse = NbrTable(km1.fwd.t, km1.fwd.n, counts=km1.fwd.counts * 0 + 1)  # 27 pairs in n rows: sparse
    sparse._pairs, sparse.wgrad_uses = None, 1
    assert not wgrad_pairs_enabled(sparse, 128, 128)  # first two uses: no list build or density read-back
    sparse.wgrad_uses = 2
    assert wgrad_pairs_enabled(sparse, 128, 128) and not wgrad_pairs_enabled(sparse, 64, 64)
    monkeypatch.setenv("FVDB_WG_PAIRS", "0")
    assert not wgrad_pairs_enabled(sparse, 128, 128)
    monkeypatch.setenv("FVDB_WG_PAIRS", "force")
    assert not wgrad_pairs_enabled(km1.fwd, 64, 64) and wgrad_pairs_enabled(km1.fwd, 64, 128)


def test_wgrad_pairs_wide_channel_blocks(maps, monkeypatch):
    """Cin = 256 is split into 128-channel blocks (conv.wgrad); each block runs the pair kernel."""
    g, go_grid, km, (ins, outs) = maps["s2"]
    rng = np.random.default_rng(3)
    x = rng.normal(size=(g.num_voxels, 256)).astype(np.float32)
    gy = rng.normal(size=(go_grid.num_voxels, 64)).astype(np.float32)
    _, gw_r = O.conv_backward(ins, outs, bf16_round(gy), bf16_round(x), np.zeros((64, 256, 3, 3, 3)))
    monkeypatch.setenv("FVDB_WG_PAIRS", "force")
    gw = wgrad(torch.from_numpy(x).cuda().to(torch.bfloat16), torch.from_numpy(gy).cuda().to(torch.bfloat16), km.fwd)
    assert tuple(gw.shape) == (64, 256, 3, 3, 3) and rel(gw, gw_r) < 2e-5
