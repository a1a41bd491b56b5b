"""Shared fixtures.  ``-m gpu`` tests need a B200 and the built libptsbe.so;
everything else runs on CPU (oracle vs golden vectors, host logic, ABI exports)."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
GOLDEN = REPO / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libptsbe.so")


@pytest.fixture(scope="session")
def golden():
    return json.loads((GOLDEN / "golden.json").read_text())


@pytest.fixture(scope="session")
def golden_arrays():
    with np.load(GOLDEN / "golden.npz") as z:
        return {k: z[k] for k in z.files}


def build_case(case, mod=None):
    """Parse a golden case with this package's parser."""
    import paper_2504_16297_b200 as P
    m = mod or P
    c = m.parse_circuit(case["circuit"])
    if case["noise"] is not None:
        c = m.attach_noise(c, m.parse_noise_model(case["noise"]))
    return c


def spec_from_json(d):
    import paper_2504_16297_b200 as P
    return P.TrajectorySpec(tuple(tuple(p) for p in d["selections"]), d["shots"], d["joint_prob"], d["tags"])


@pytest.fixture(scope="session")
def libptsbe():
    """Path of the built shared library (built here with nvcc if missing)."""
    from paper_2504_16297_b200 import build
    return build.build()
