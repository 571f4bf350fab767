"""Golden P1 element matrices from the REFERENCE:
assemble_mass / assemble_stiffness (quadrature assembly, fem/assembly.hpp:81-161),
lumped_mass_vector (:241-262) and apply_constraints_precision_pair with
embed_dirichlet (fem/constraints.hpp:158-173, priors/boundary.hpp:15-29), for the
config-4 slice (999 elements on [-1, 1], Burgers proxy ν = 0.01/π, c = 0.5), the
config-1 slice (999 elements on [0, 1]) and a config-2/5-shaped unit square
(31² cells, heat proxy ε² = 0.0025). TEST INFRASTRUCTURE; run in the build
container: python tests/golden/make_golden_fem.py -> tests/golden/fem_p1.npz
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle.pyoracle import Ref  # noqa: E402

CASES = {
    "c4": [1, 999, -1.0, 1.0, 0.01 / np.pi, 0.5, 0.0, 1, 1e-10],
    "c1": [1, 999, 0.0, 1.0, 1.0, 0.0, 400.0, 0, 0.0],
    "sq": [2, 31, 0.0, 1.0, 0.0025, 0.0, 0.0, 0, 0.0],
}

out = {}
ref = Ref()
for name, p in CASES.items():
    b = ref.build("fem", p)
    out[name + "_params"] = np.array(p, np.float64)
    for m in ["M", "K"] + (["M_c", "K_c"] if p[7] else []):
        a = b.mat(m)
        out[f"{name}_{m}_cp"] = np.asarray(a.col_ptr, np.int64)
        out[f"{name}_{m}_ri"] = np.asarray(a.row_idx, np.int32)
        out[f"{name}_{m}_v"] = np.asarray(a.values, np.float64)
    out[name + "_lumped"] = b.vec("lumped")
    if p[7]:
        out[name + "_lumped_c"] = b.vec("lumped_c")
np.savez_compressed(os.path.join(HERE, "fem_p1.npz"), **out)
print({k: v.shape for k, v in out.items()})
