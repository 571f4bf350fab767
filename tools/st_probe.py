import sys, time, json, math
import numpy as np
sys.path.insert(0, '.')
from paper_2503_08343_b200.spacetime import SpaceTimePosterior, SpaceTimeSpec, GaussNewtonConfig
which = sys.argv[1] if len(sys.argv) > 1 else "c4"
spec = SpaceTimeSpec.burgers() if which == "c4" else SpaceTimeSpec.heat()
t = time.perf_counter(); post = SpaceTimePosterior(spec); tc = time.perf_counter() - t
x = spec.node_x()
if which == "c4":
    u0 = -np.sin(np.pi * x)
else:
    from oracle.pyoracle import Ref
    rng = np.random.default_rng(0); a = rng.standard_normal(10) / np.arange(1, 11)
    u0 = sum(a[k-1] * np.sin(k * np.pi * x) for k in range(1, 11))
for rep in range(2):
    t = time.perf_counter(); mean, var, trace, conv = post.run(u0, variances=True); tr = time.perf_counter() - t
    i = post.info()
    print(json.dumps(dict(which=which, rep=rep, create_s=tc, run_s=tr, n=i.n, nnz_pat=i.nnz_pattern, nnz_l=i.nnz_l, nnz_l_pad=i.nnz_l_padded,
        flops=i.flops_ref, flops_sn=i.flops_sn, setup_host_ms=i.setup_host_ms, assemble_ms=i.assemble_ms, condition_ms=i.condition_ms,
        gn_ms=i.gn_ms, laplace_ms=i.laplace_ms, selinv_ms=i.selinv_ms, numeric_ms=i.numeric_ms, nfac=i.n_factorizations,
        launches=i.kernel_launches, trace=[(t.objective, t.decrement, t.step_size, t.backtracks) for t in trace],
        mean_norm=float(np.linalg.norm(mean)), var_min=float(var.min()), var_max=float(var.max()))), flush=True)
