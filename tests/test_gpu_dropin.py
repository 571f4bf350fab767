"""Drop-in proof: the reference's own acceptance suite (tests/acceptance.cpp,
unmodified) compiled with paper_2503_08343_b200/include first on the include
path, so every cholesky_factor / solve_triangular / takahashi_* call the
reference makes (gmrf.hpp, gauss_newton.hpp, spatiotemporal.hpp, the tests)
runs on the GPU through include/gmrf_b200.h. Built by `make -C oracle dropin`
where /root/reference exists; the binary travels to the GPU box."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")


def test_reference_acceptance_suite_on_gpu():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/acceptance_b200 not built (reference absent at build time)")
    out = subprocess.run([BIN], cwd=os.path.dirname(BIN), capture_output=True, text=True,
                         timeout=900)
    lines = [ln for ln in out.stdout.splitlines() if "criterion-" in ln]
    assert len(lines) == 10, out.stdout + out.stderr
    for crit in (1, 2, 10):  # the factor / solve / Takahashi criteria
        assert any(ln.startswith(f"PASS criterion-{crit}:") for ln in lines), out.stdout
    assert out.returncode == 0, out.stdout
