"""GPU: signature-sorted neighbour tables for the gather-GEMM kernel (fvdb_kmap_signature_order,
fvdb_conv_gather_tc_perm in csrc/conv_tc.cu).

Sorting output rows by their 27-bit offset signature is a pure re-ordering: each output row still
sums the same pairs in the same offset order, so the permuted conv must equal the unpermuted one
(bitwise) and the oracle (conv.py:180-191 / 358-366 forms, bf16-rounded inputs, rel <= 2e-5).
"""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2407_01781_b200 as P
from paper_2407_01781_b200.conv import gather_conv, pack_weights_umma
from paper_2407_01781_b200.workloads import sphere_shell_coords

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = a.detach().double().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def bf16_round(a):
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).float().numpy().astype(np.float64)


@pytest.fixture
def sig_sort(monkeypatch):
    def set_(on):
        monkeypatch.setenv("FVDB_SIG_SORT", "force" if on else "0")
    return set_


@pytest.fixture(scope="module")
def maps():
    c = sphere_shell_coords(40, band=1.5)
    g, _ = P.build_from_coords(c)
    og = O.build_from_coords(c)
    gc, ogc = P.coarsen(g, 2), O.coarsen(og, 2)
    km2 = P.build_kernel_map(g, gc, 2)
    ins2, outs2 = O.kernel_map(og, ogc, 2)
    km1 = P.build_kernel_map(g, g, 1)
    ins1, outs1 = O.kernel_map(og, og, 1)
    return g, gc, (km1, ins1, outs1), (km2, ins2, outs2)


@pytest.mark.parametrize("which", ["s1_fwd", "s2_fwd", "s2_bwd"])
def test_signature_order_is_stable_sort(maps, which):
    _, _, (km1, _, _), (km2, _, _) = maps
    tab = {"s1_fwd": km1.fwd, "s2_fwd": km2.fwd, "s2_bwd": km2.bwd}[which]
    tp, perm, masks = tab.signature_sorted()
    v = tab.view.cpu().numpy()
    sig = ((v >= 0).astype(np.int64) << np.arange(27)[:, None]).sum(0)
    expect = np.argsort(sig, kind="stable")
    assert np.array_equal(perm[:tab.n].cpu().numpy(), expect)
    tpn = tp.cpu().numpy()
    assert np.array_equal(tpn[:, :tab.n], v[:, expect])
    assert (tpn[:, tab.n:] == -1).all()
    check_masks(masks, tpn, tab.n)
    check_masks(tab.tile_masks(), v, tab.n)


def check_masks(masks, table, n):
    """masks[t] bit d == some row of 128-row tile t has a pair at offset d."""
    has = table[:, :n] >= 0
    pad = (-n) % 128
    has = np.pad(has, ((0, 0), (0, pad))).reshape(27, -1, 128).any(-1)
    expect = (has.astype(np.int64) << np.arange(27)[:, None]).sum(0)
    assert np.array_equal(masks.cpu().numpy().astype(np.int64) & ((1 << 27) - 1), expect)


@pytest.mark.parametrize("K,N", [(32, 32), (64, 64), (64, 128), (128, 64)])
def test_sorted_gather_equals_unsorted_and_oracle(maps, sig_sort, K, N):
    g, gc, _, (km, ins, outs) = maps
    rng = np.random.default_rng(K + 3 * N)
    x = rng.normal(size=(g.num_voxels, K)).astype(np.float32)
    w = (rng.normal(size=(N, K, 3, 3, 3)) / np.sqrt(27 * K)).astype(np.float32)
    gy = rng.normal(size=(gc.num_voxels, N)).astype(np.float32)
    xb, gyb, wt = (torch.from_numpy(a).cuda() for a in (x, gy, w))
    xb, gyb = xb.to(torch.bfloat16), gyb.to(torch.bfloat16)
    res = {}
    for on in (False, True):
        sig_sort(on)
        res[on] = (gather_conv(xb, km.fwd, wt, out_dtype=torch.float32, impl="gather"),
                   gather_conv(gyb, km.bwd, wt, transpose=True, out_dtype=torch.float32, impl="gather"),
                   gather_conv(xb, km.fwd, wt, impl="gather"))
    for a, b in zip(res[False], res[True]):
        assert torch.equal(a, b)
    y, gi, _ = res[True]
    assert rel(y, O.conv_igemm(bf16_round(x), bf16_round(w), ins, outs, gc.num_voxels)) < 2e-5
    gi_r, _ = O.conv_backward(ins, outs, bf16_round(gy), bf16_round(x), bf16_round(w))
    assert rel(gi, gi_r) < 2e-5


def test_policy_sorts_sparse_tables_only(maps, monkeypatch):
    from paper_2407_01781_b200.conv import sig_sort_enabled
    _, _, (km1, _, _), (km2, _, _) = maps
    monkeypatch.delenv("FVDB_SIG_SORT", raising=False)
    assert sig_sort_enabled(km2.bwd) and km2.bwd.sparse  # transposed stride-2 table: sorted by default
    assert not sig_sort_enabled(km2.fwd) and not sig_sort_enabled(km1.fwd)
    monkeypatch.setenv("FVDB_SIG_SORT", "1")
    assert km2.bwd.density() < 5 and sig_sort_enabled(km2.bwd)
    assert km1.fwd.density() > 15 and not sig_sort_enabled(km1.fwd)


def test_sorted_tiny_and_empty(sig_sort):
    sig_sort(True)
    g, _ = P.build_from_coords(np.array([[0, 0, 0], [5, 5, 5]]))
    km = P.build_kernel_map(g, g, 1)
    x = torch.ones(2, 64, device="cuda", dtype=torch.bfloat16)
    w = torch.ones(64, 64, 3, 3, 3, device="cuda") / 64
    y = gather_conv(x, km.fwd, w, out_dtype=torch.float32, impl="gather")
    assert torch.allclose(y, torch.ones_like(y))
    ge = P.build_from_coords(np.zeros((0, 3), np.int64))[0]
    kme = P.build_kernel_map(ge, ge, 1)
    ye = gather_conv(torch.zeros(0, 64, device="cuda", dtype=torch.bfloat16), kme.fwd, w, impl="gather")
    assert ye.shape == (0, 64)


def test_masked_gather_equals_unmasked_and_oracle(maps, sig_sort):
    """Tile masks only drop (super-tile, offset) stages without pairs: results are bitwise those of the
    unmasked kernel (fvdb_conv_gather_tc), sorted or not, and match the oracle."""
    from paper_2407_01781_b200 import _lib
    g, gc, (km1, ins1, outs1), (km2, ins2, outs2) = maps
    rng = np.random.default_rng(5)
    for tab, K, N, tr, n_in, ref_fn in (
            (km1.fwd, 64, 64, False, g.num_voxels,
             lambda x, w: O.conv_igemm(bf16_round(x), bf16_round(w), ins1, outs1, g.num_voxels)),
            (km2.bwd, 128, 64, True, gc.num_voxels,
             lambda x, w: O.conv_backward(ins2, outs2, bf16_round(x), np.zeros((g.num_voxels, 64)),
                                          bf16_round(w))[0])):
        x = rng.normal(size=(n_in, K)).astype(np.float32)
        w = (rng.normal(size=((K, N) if tr else (N, K)) + (3, 3, 3)) / np.sqrt(27 * K)).astype(np.float32)
        xb, wt = torch.from_numpy(x).cuda().to(torch.bfloat16), torch.from_numpy(w).cuda()
        img = pack_weights_umma(wt, tr, "gather")
        plain = torch.empty((tab.n, N), dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib().fvdb_conv_gather_tc(xb.data_ptr(), n_in, K, img.data_ptr(), N, tab.t.data_ptr(), tab.ld,
                                                  tab.n, plain.data_ptr(), _lib.DTYPE_F32, _lib.stream_ptr()), "plain")
        for on in (False, True):
            sig_sort(on)
            y = gather_conv(xb, tab, wt, transpose=tr, out_dtype=torch.float32, w_image=img)
            assert torch.equal(y, plain)
        assert rel(plain, ref_fn(x, w)) < 2e-5
