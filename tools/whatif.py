"""Timing what-if for one config-4 factorization (GMRF_WHATIF bitmask skips
launch classes: 1 trailing GEMM rest, 2 panels, 4 next-block GEMM, 8 extend-add).
Results are numerically invalid; only the replayed-graph time is meaningful."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2503_08343_b200.spacetime import SpaceTimePosterior, SpaceTimeSpec, GaussNewtonConfig
spec = SpaceTimeSpec.burgers()
post = SpaceTimePosterior(spec, GaussNewtonConfig(max_iters=1))
u0 = -np.sin(np.pi * spec.node_x())
ts, sv = [], []
var = len(sys.argv) > 1 and sys.argv[1] == "var"
for rep in range(4):
    try:
        post.run(u0, variances=var, copy_back=False)
    except Exception as e:  # noqa: BLE001
        pass
    i = post.info()
    ts.append(i.numeric_ms / max(1, i.n_factorizations))
    sv.append(i.selinv_ms)
print("per-factorization ms", [round(t, 3) for t in ts], "selinv ms", [round(t, 3) for t in sv])
