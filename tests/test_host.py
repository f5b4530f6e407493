"""CPU: the C-ABI library loads and exports its header; host-side validation and errors."""
import ctypes
import pathlib
import re

import numpy as np
import pytest
import torch

import paper_2407_01781_b200 as P
from paper_2407_01781_b200 import _lib
from paper_2407_01781_b200.dist import partition_by_cost

HEADER = pathlib.Path(__file__).resolve().parents[1] / "include" / "fvdb_b200.h"


def header_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(fvdb_\w+)\(", text, re.M)))


def test_library_exports_every_header_symbol():
    h = _lib.load_library()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(h, s), s
        assert s in _lib.SIGNATURES, f"{s} missing from the ctypes binding"
    assert set(_lib.SIGNATURES) == set(syms)
    assert h.fvdb_version().startswith(b"fvdb_b200")


def test_library_is_sm100a():
    so = _lib.LIB_PATH.read_bytes()
    assert b"sm_100a" in so


def test_workspace_queries_need_no_gpu():
    h = _lib.load_library()
    assert h.fvdb_build_workspace_bytes(1000) > 8 * 1000 * 6
    assert h.fvdb_kmap_workspace_bytes(10) >= 27 * 10 * 4
    assert h.fvdb_kmap_compact_workspace_bytes(100) > 27 * 100 * 8
    assert h.fvdb_wgrad_workspace_bytes(0, 1000, 8, 16) >= 27 * 8 * 16 * 4


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    with pytest.raises(_lib.FvdbError, match="no CPU fallback"):
        P.build_from_coords(np.zeros((4, 3), np.int64))


def test_conv_kernel_validation():
    with pytest.raises(ValueError):
        P.ConvKernel(np.ones((2, 2, 3, 3)))
    with pytest.raises(ValueError):
        P.ConvKernel(np.full((1, 1, 3, 3, 3), np.nan))
    k = P.ConvKernel.identity(4)
    assert k.c_in == 4 and k.c_out == 4 and float(k.spoke(0, 0, 0).trace()) == 4.0


def test_kernel_map_stride_rejected_before_device_work():
    with pytest.raises(ValueError, match="stride"):
        P.build_kernel_map(None, None, 3)


def test_offset_index_and_stencil():
    assert P.KernelMap.offset_index(-1, -1, -1) == 0
    assert P.KernelMap.offset_index(0, 0, 0) == 13
    assert P.KernelMap.offset_index(1, 1, 1) == 26
    assert P.STENCIL.shape == (27, 3) and (P.STENCIL[13] == 0).all()
    for d, (a, b, c) in enumerate(P.STENCIL):
        assert P.KernelMap.offset_index(a, b, c) == d


def test_jagged_layout_and_errors():
    jt = P.jagged_from_list([np.ones((2, 3)), np.zeros((0, 3)), np.ones((4, 3))])
    assert jt.joffsets.tolist() == [[0, 2], [2, 2], [2, 6]]
    assert jt.jidx.tolist() == [0, 0, 2, 2, 2, 2]
    assert [e.shape[0] for e in jt.unbind()] == [2, 0, 4]
    with pytest.raises(ValueError, match="trailing shape"):
        P.jagged_from_list([np.ones((2, 3)), np.ones((2, 4))])
    with pytest.raises(ValueError, match="at least one"):
        P.jagged_from_list([])
    with pytest.raises(ValueError, match="tile"):
        P.JaggedTensor(np.ones((3, 1)), [[0, 2]], [0, 0, 0])
    with pytest.raises(ValueError, match="jidx"):
        P.JaggedTensor(np.ones((2, 1)), [[0, 2]], [0, 1])
    with pytest.raises(ValueError, match="row count"):
        jt.with_data(np.ones((5, 3)))


def test_grid_batch_requires_grids_and_type_checks():
    with pytest.raises(ValueError):
        P.GridBatch([])
    with pytest.raises(TypeError, match="GridBatch"):
        P.conv_batch([1, 2], np.ones((1, 1)), np.ones((1, 1, 3, 3, 3)))


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition_by_cost_is_contiguous_cover(world):
    rng = np.random.default_rng(world)
    costs = rng.integers(1, 100, size=13).tolist()
    parts = partition_by_cost(costs, world)
    assert len(parts) == world
    assert parts[0][0] == 0 and parts[-1][1] == len(costs)
    for (a, b), (c, d) in zip(parts, parts[1:]):
        assert b == c and a <= b
    if world <= len(costs):
        loads = [sum(costs[a:b]) for a, b in parts]
        assert max(loads) <= sum(costs) / world + max(costs)


def test_choose_variant_thresholds_match_reference():
    class G:
        def __init__(self, occ):
            self.o = occ

        def leaf_occupancy(self):
            return self.o

    assert P.choose_variant(G(1.0), 64, 64) == "brick"
    assert P.choose_variant(G(0.1), 128, 128) == "lggs"
    assert P.choose_variant(G(0.1), 8, 16) == "igemm"
    assert P.choose_variant(G(0.3), 32, 32) == "leaf"
    assert P.choose_variant(G(0.3), 64, 64) == "igemm"


def _table(n, pairs_per_row, sparse=False):
    from paper_2407_01781_b200.conv import NbrTable
    t = NbrTable(torch.full((27, 512), -1, dtype=torch.int32), n,
                 counts=torch.full((27,), int(round(pairs_per_row * n / 27)), dtype=torch.int64))
    t.sparse = sparse
    return t


def test_conv_kernel_policy_host_logic(monkeypatch):
    """steady_impl / sig_sort_enabled (conv.py): the kernel a reused table settles on, from its density, the
    layer width and the sparse flag (transposed stride-2 tables); FVDB_SIG_SORT overrides."""
    from paper_2407_01781_b200.conv import HALO_MIN_DENSITY_WIDE, sig_sort_enabled, steady_impl
    monkeypatch.delenv("FVDB_SIG_SORT", raising=False)
    dense, lidar = _table(270, 20.85), _table(270, 9.23)
    assert steady_impl(dense, 64, 64) == ("halo", False)
    assert steady_impl(dense, 64, 128) == ("halo", False)         # dense wide layer: halo
    assert steady_impl(lidar, 64, 64) == ("halo", False)          # sparse narrow layer: halo
    assert steady_impl(lidar, 128, 128) == ("gather", True)       # sparse wide layer: sorted gather
    assert steady_impl(_table(270, HALO_MIN_DENSITY_WIDE - 1), 64, 128) == ("gather", True)
    sp = _table(270, 3.1, sparse=True)
    assert sig_sort_enabled(sp) and steady_impl(sp, 128, 64) == ("gather", True)
    assert not sig_sort_enabled(lidar)
    monkeypatch.setenv("FVDB_SIG_SORT", "0")
    assert not sig_sort_enabled(sp)
    monkeypatch.setenv("FVDB_SIG_SORT", "1")
    assert sig_sort_enabled(lidar) and not sig_sort_enabled(dense)
    monkeypatch.setenv("FVDB_SIG_SORT", "force")
    assert sig_sort_enabled(dense)


def test_exact_skip_policy(monkeypatch):
    """fp32 / f64 gather: plain table on first use, signature-sorted from the second use (tiled shapes)."""
    import torch
    from paper_2407_01781_b200.conv import NbrTable, exact_skip_mode
    monkeypatch.delenv("FVDB_EXACT_SKIP", raising=False)
    t = NbrTable(torch.full((27, 128), -1, dtype=torch.int32), 10)
    assert exact_skip_mode(t, 32, 32) == "none"
    t.exact_uses = 1
    assert exact_skip_mode(t, 32, 32) == "sort"
    assert exact_skip_mode(t, 32, 128) == "none"  # N > 64: untiled kernel, no row permutation
    monkeypatch.setenv("FVDB_EXACT_SKIP", "sort")
    assert exact_skip_mode(t, 32, 128) == "masks"


def test_nbr_table_lazy_construction():
    """NbrTable(t=callable, ld=...): the table is built once, on the first read of .t (a same-grid map's transposed
    table: the halo dgrad runs the forward plan reversed and never reads it; conv.py KernelMap.bwd)."""
    from paper_2407_01781_b200.conv import NbrTable
    calls = []
    base = torch.arange(27 * 256, dtype=torch.int32).reshape(27, 256)

    def make():
        calls.append(1)
        return torch.flip(base, dims=[0])

    t = NbrTable(make, 200, ld=256)
    assert t.ld == 256 and t.n == 200 and not calls  # shape known, nothing built
    assert torch.equal(t.t, torch.flip(base, dims=[0])) and len(calls) == 1
    assert t.t is t.t and len(calls) == 1            # cached
    eager = NbrTable(base, 200)
    assert eager.ld == 256 and eager.t is base
