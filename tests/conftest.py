"""Shared fixtures. Markers: ``gpu`` = needs a CUDA device (B200)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA device (runs on the B200 box)")


@pytest.fixture(scope="session")
def port():
    from oracle.pyoracle import Port
    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle.pyoracle import Ref
    if not Ref.available():
        pytest.skip("oracle/_ref not built (reference absent)")
    return Ref()


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name))


def golden_mat(z, prefix):
    from paper_2503_08343_b200 import SparseMatrixCSC
    nr, nc = z[f"{prefix}_shape"]
    return SparseMatrixCSC.from_arrays(nr, nc, z[f"{prefix}_cp"], z[f"{prefix}_ri"],
                                       z[f"{prefix}_v"])


@pytest.fixture(scope="session")
def lib_built():
    from paper_2503_08343_b200 import build
    build.build()
    return True
