"""GPU: FVDBIDX1 grid files (paper_2407_01781_b200.io) against files written by the reference itself.

Bytes written by our save_grid must equal the reference writer's (io.py:40-70) and files the reference
wrote must load into identical topology arrays; corrupted files raise GridFileError with the reference's
messages (tests/golden/make_golden_io.py records them).
"""
import json

import numpy as np
import pytest

import paper_2407_01781_b200 as P
from paper_2407_01781_b200.io import GridFileError, load_grid, save_grid
from conftest import FIELDS, GOLDEN

pytestmark = pytest.mark.gpu
IO = GOLDEN / "io"
META = json.loads((IO / "meta.json").read_text())


@pytest.mark.parametrize("case", ["scattered", "multi_tile", "named_shell"])
def test_roundtrip_bytes_and_arrays(tmp_path, case):
    m = META[case]
    coords = np.load(IO / f"{case}_coords.npy")
    g, _ = P.build_from_coords(coords, P.VoxelTransform(np.array(m["voxel_size"]), np.array(m["origin"])),
                               m["name"])
    out = tmp_path / "g.fvdb"
    n = save_grid(g, out)
    ref = (IO / f"{case}.fvdb").read_bytes()
    assert n == len(ref) and out.read_bytes() == ref, "bytes differ from the reference writer"
    h = load_grid(IO / f"{case}.fvdb")
    assert h.counts == tuple(m["counts"]) and h.name == m["name"]
    assert np.allclose(h.transform.voxel_size, m["voxel_size"]) and np.allclose(h.transform.origin, m["origin"])
    a, b = g.to_numpy(), h.to_numpy()
    for f in FIELDS:
        assert np.array_equal(a[f], b[f]), f
    # the loaded grid is fully functional on the device (probes use the rebuilt keys / origins)
    idx = h.coord_to_index_many(coords)
    assert np.array_equal(np.sort(idx.cpu().numpy()), np.arange(1, h.num_voxels + 1))


def test_empty_grid(tmp_path):
    h = load_grid(IO / "empty.fvdb")
    assert h.counts == (0, 0, 0, 0) and h.name == "empty"
    out = tmp_path / "e.fvdb"
    save_grid(h, out)
    assert out.read_bytes() == (IO / "empty.fvdb").read_bytes()


@pytest.mark.parametrize("bad", sorted(META["errors"]))
def test_corrupted_files_match_reference_errors(bad):
    msg = META["errors"][bad]
    with pytest.raises(GridFileError) as ei:
        load_grid(IO / f"{bad}.fvdb")
    assert isinstance(ei.value, ValueError)
    assert str(ei.value) == msg
