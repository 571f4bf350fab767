"""Small driver for ncu captures: config-4-shaped posterior at reduced size, 1 GN step."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2503_08343_b200.spacetime import SpaceTimePosterior, SpaceTimeSpec, GaussNewtonConfig
n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 499
n_t = int(sys.argv[2]) if len(sys.argv) > 2 else 500
spec = SpaceTimeSpec.burgers(n_el=n_el, n_t=n_t)
post = SpaceTimePosterior(spec, GaussNewtonConfig(max_iters=1))
u0 = -np.sin(np.pi * spec.node_x())
post.run(u0, variances=True, copy_back=False)
print("ok", post.info().numeric_ms)
