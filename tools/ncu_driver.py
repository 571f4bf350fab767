"""One config-4 posterior (1 GN step) for ncu captures: python tools/ncu_driver.py [n_el n_t]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2503_08343_b200.spacetime import GaussNewtonConfig, SpaceTimePosterior, SpaceTimeSpec  # noqa: E402

n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 999
n_t = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
spec = SpaceTimeSpec.burgers(n_el, n_t)
post = SpaceTimePosterior(spec, GaussNewtonConfig(max_iters=1))
post.run(-np.sin(np.pi * spec.node_x()), variances=True, copy_back=False)
