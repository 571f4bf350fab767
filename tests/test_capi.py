"""The C-ABI library loads and exports every symbol include/gmrf_b200.h declares;
without a GPU the numeric entry points fail loudly (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "gmrf_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gmrf_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(lib_built):
    from paper_2503_08343_b200 import _capi
    lib = C.CDLL(_capi.LIB_PATH)
    names = _declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
        assert name in _capi.SIGNATURES, f"{name} missing from the ctypes table"


def test_no_cpu_fallback(lib_built):
    import numpy as np
    import torch
    import paper_2503_08343_b200 as g
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    q = g.SparseMatrixCSC.from_arrays(2, 2, [0, 2, 4], [0, 1, 0, 1], [4.0, 2.0, 2.0, 3.0])
    with pytest.raises(g.DeviceError):
        g.cholesky_factor(q, np.arange(2))


def test_rng_mirror_matches_reference_draws(lib_built, ref):
    """gmrf_rng_fill reproduces core/rng.hpp: the reference's sample_direct on
    Q = I, μ = 0 returns its z draws verbatim (gmrf.hpp:173-184)."""
    import numpy as np
    import scipy.sparse as sp
    import paper_2503_08343_b200 as g
    n = 9
    q = sp.eye(n).tocsc()
    x = ref.sample_direct(n, q.indptr, q.indices, q.data, np.arange(n), np.zeros(n), 3, 2002)
    assert np.array_equal(x.ravel(order="F"), g.Rng(2002).normal_vector(3 * n))
    u = g.Rng(1001).uniforms(5)
    assert np.all((u > 0) & (u < 1))
