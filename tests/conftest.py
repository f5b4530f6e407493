import json
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200, sm_100a) device")
    config.addinivalue_line("markers", "slow: full-size configuration")


def _npz(name):
    with np.load(GOLDEN / name) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_grids():
    return _npz("grids.npz")


@pytest.fixture(scope="session")
def golden_kmaps():
    return _npz("kmaps.npz")


@pytest.fixture(scope="session")
def golden_convs():
    return _npz("convs.npz")


@pytest.fixture(scope="session")
def golden_fixtures():
    return _npz("fixtures_ref.npz")


@pytest.fixture(scope="session")
def golden_sizes():
    return json.loads((GOLDEN / "sizes.json").read_text())


GRID_CASES = ("scattered", "dup_heavy", "single", "pair", "multi_tile", "wide", "neg_boundary", "shell",
              "small_shell", "clustered")
KMAP_CASES = ("scattered", "shell", "clustered", "multi_tile", "neg_boundary", "pair")
CONV_CASES = ("scattered", "small_shell", "clustered")
FIELDS = ("tile_keys", "upper_origins", "upper_child_starts", "lower_offset_in_upper", "lower_origins",
          "lower_child_starts", "leaf_offset_in_lower", "leaf_keys", "leaf_origins", "leaf_masks",
          "leaf_prefix", "leaf_value_offset")
