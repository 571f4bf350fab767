"""Dumps the product's full-size config-4 GN trace, mode and variances (n = 1e6) to
gpurun_out/c4_full_gpu.npz, for the reverse parity probe of tests/golden/make_golden_full.py
(order_novar:/floor_novar: compare the unmodified reference's run against a fixture-shaped file)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2503_08343_b200.spacetime import GaussNewtonConfig, SpaceTimePosterior, SpaceTimeSpec  # noqa: E402

spec = SpaceTimeSpec.burgers()
post = SpaceTimePosterior(spec, GaussNewtonConfig(max_iters=10))
mean, var, trace, conv = post.run(-np.sin(np.pi * spec.node_x()), variances=True)
np.savez_compressed(os.path.join(ROOT, "gpurun_out", "c4_full_gpu.npz"), mode=mean, var_post=var,
                    gn_objective=np.array([t.objective for t in trace]),
                    gn_decrement=np.array([t.decrement for t in trace]),
                    gn_step=np.array([t.step_size for t in trace]),
                    gn_backtracks=np.array([float(t.backtracks) for t in trace]),
                    gn_converged=np.array(float(conv)))
print([(t.objective, t.decrement, t.step_size, t.backtracks) for t in trace], conv)
