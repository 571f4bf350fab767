"""The scheduling / kernel variants of the factorization must not change a bit.

Each variant below only changes WHERE or WITH WHICH tile shape a product is
computed, never the per-entry summation order: deferred (K = 256) against right-looking
(K = 64) trailing updates, the 32×32 chain GEMM (k_gemm_next) against the 64×64
one, the update-block extend-add on the bulk stream, the CTA-per-column
extend-add. (The 128×128 TMA-staged GEMM agrees bit for bit with the 64×64 one
per launch, tools/gemm_big_bench.cu; inside a factorization it also replaces
split-K launches, so it is compared to rounding.) The knobs are read when a factor is created, so one process can
build the same posterior under two settings and compare the results exactly.

The config-5 shape used here (48² nodes × 96 slices, n = 221,184) is the
smallest whose top separators (2304 unknowns) reach the wide kernel's and the
deferral's thresholds; the small golden fixtures never do.
"""
import os

import numpy as np
import pytest

from paper_2503_08343_b200.spacetime import GaussNewtonConfig, SpaceTimePosterior, SpaceTimeSpec

pytestmark = pytest.mark.gpu


def _run(spec, u0, env, gn=1):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        post = SpaceTimePosterior(spec, GaussNewtonConfig(max_iters=gn))
        mean, var, trace, _ = post.run(u0, variances=True)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return mean, var, [(t.objective, t.decrement, t.step_size, t.backtracks) for t in trace]


def _same(a, b):
    assert a[2] == b[2]
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])


def _close(a, b, tol=1e-9):
    # same Gauss-Newton path (steps, backtracks), values to rounding
    assert [t[2:] for t in a[2]] == [t[2:] for t in b[2]]
    for x, y in zip(a[2], b[2]):
        assert abs(x[0] - y[0]) <= 1e-8 * abs(y[0]) and abs(x[1] - y[1]) <= 1e-6 * abs(y[1])
    assert np.linalg.norm(a[0] - b[0]) <= tol * np.linalg.norm(b[0])
    assert np.linalg.norm(a[1] - b[1]) <= tol * np.linalg.norm(b[1])


def test_wide_gemm_and_deferral_on_large_fronts():
    """On this shape the 64×64 path splits the K of its closing SYRKs (too few
    tiles to fill the GPU) while the 128×128 tiles never split, so the two differ
    by rounding only; deferral keeps the summation order and must match exactly."""
    spec = SpaceTimeSpec.allen_cahn(47, 96)
    u0 = np.random.default_rng(1005).uniform(-0.1, 0.1, spec.n_space)
    base = _run(spec, u0, {})
    assert np.all(np.isfinite(base[0])) and np.all(base[1] > 0)
    _close(base, _run(spec, u0, {"GMRF_WIDE_K": "0"}))  # 64×64 tiles everywhere
    _same(base, _run(spec, u0, {"GMRF_DEFER": "1"}))    # plain right-looking updates


@pytest.mark.parametrize("env", [{"GMRF_GEMM_NEXT": "0"}, {"GMRF_EA_SPLIT": "0"},
                                 {"GMRF_EA_CTA": "0"}, {"GMRF_EA_CTA": "1000000"}])
def test_chain_variants_are_bit_identical(env):
    spec = SpaceTimeSpec.burgers(299, 300)
    u0 = -np.sin(np.pi * spec.node_x())
    _same(_run(spec, u0, {}, gn=2), _run(spec, u0, env, gn=2))


@pytest.mark.parametrize("shape", ["burgers", "allen_cahn"])
def test_blocked_selected_inversion_matches_chunk_chain(shape):
    """The blocked selected inversion (W = L_JJ⁻¹ by recursive doubling, then
    Gn = −L_RJ W, Σ_RJ = Σ_RR Gn, Σ_JJ = WᵀW + GnᵀΣ_RJ as GEMM stages; selinv.cuh)
    and the 64-column chunk chain (GMRF_SEL_BLOCK=0) evaluate the same Takahashi
    recurrences (takahashi.hpp:43-60) in different association orders: the
    factorization, mean and GN trace must be untouched, the variances agree to
    rounding amplified by the conditioning of the diagonal blocks."""
    if shape == "burgers":
        spec = SpaceTimeSpec.burgers(299, 300)
        u0 = -np.sin(np.pi * spec.node_x())
    else:
        spec = SpaceTimeSpec.allen_cahn(31, 64)
        u0 = np.random.default_rng(1005).uniform(-0.1, 0.1, spec.n_space)
    blocked = _run(spec, u0, {}, gn=2)
    chain = _run(spec, u0, {"GMRF_SEL_BLOCK": "0"}, gn=2)
    only_wide = _run(spec, u0, {"GMRF_SEL_BLOCK_MIN": "65"}, gn=2)
    for other in (chain, only_wide):
        assert blocked[2] == other[2]
        np.testing.assert_array_equal(blocked[0], other[0])
        assert np.all(other[1] > 0)
        rel = np.abs(blocked[1] - other[1]) / other[1]
        assert rel.max() <= 1e-9, rel.max()


def test_inverted_wide_blocks_match_substitution():
    """Wide supernodes end each 64-row block step of the solves with a GEMV against
    the inverted diagonal block (k_tri_inv64 after every factorization) instead of
    a 64-step warp substitution (GMRF_WIDE_INV=0): same Gauss-Newton path, values
    to rounding."""
    spec = SpaceTimeSpec.burgers(299, 300)
    u0 = -np.sin(np.pi * spec.node_x())
    _close(_run(spec, u0, {}, gn=3), _run(spec, u0, {"GMRF_WIDE_INV": "0"}, gn=3), tol=1e-8)
