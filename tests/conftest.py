"""Shared fixtures.  ``-m gpu`` tests need a B200 and the built CUDA library;
everything else runs on CPU (oracle vs golden vectors, host logic, C-ABI
export checks, gloo multi-process tests)."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built libdiffproj_b200.so")


def load_golden(name):
    d = np.load(os.path.join(GOLDEN, name), allow_pickle=False)
    return {k: d[k] for k in d.files}


@pytest.fixture
def rng():
    return np.random.default_rng(0)


SCENES = ["bar_arap", "bar_neohookean", "hanging_sheet", "block_on_plane",
          "friction_high", "friction_ident", "block_lift", "single_tet_nh",
          "cube2_slide", "c1lite", "c1"]
