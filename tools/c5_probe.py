"""Config-5 (Allen-Cahn, 2-D unit square × time) at several sizes on one GPU."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from paper_2503_08343_b200.spacetime import SpaceTimePosterior, SpaceTimeSpec, GaussNewtonConfig
for arg in sys.argv[1:]:
    nc, nt = map(int, arg.split("x"))
    spec = SpaceTimeSpec.allen_cahn(n_cells=nc, n_t=nt)
    t0 = time.time()
    try:
        post = SpaceTimePosterior(spec, GaussNewtonConfig(max_iters=8))
    except Exception as e:
        print(arg, "setup failed:", str(e)[:200], flush=True)
        continue
    i = post.info()
    print(arg, "n", i.n, "nnz_l %.3e" % i.nnz_l, "flops %.3e" % i.flops_sn, "setup %.1fs" % (time.time() - t0), flush=True)
    rng = np.random.default_rng(1005)
    u0 = -0.1 + 0.2 * rng.random(spec.n_space)
    for rep in range(2):
        t0 = time.time()
        mean, var, trace, conv = post.run(u0, variances=True, copy_back=False)
        dt = time.time() - t0
    i = post.info()
    print(arg, "run %.3fs" % dt, "iters", len(trace), "conv", conv, "numeric ms/fact %.2f" % (i.numeric_ms / i.n_factorizations),
          "TF/s %.2f" % (i.flops_sn / (i.numeric_ms / i.n_factorizations) / 1e9), "selinv %.1f ms" % i.selinv_ms, flush=True)
