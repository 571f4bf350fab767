"""Per-level solve profile of the config-4 factor: time, algorithmic bytes, GB/s."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2503_08343_b200.spacetime import SpaceTimePosterior, SpaceTimeSpec, GaussNewtonConfig
spec = SpaceTimeSpec.burgers()
post = SpaceTimePosterior(spec, GaussNewtonConfig(max_iters=1))
u0 = -np.sin(np.pi * spec.node_x())
post.run(u0, variances=True, copy_back=False)
post.set_profile(2)
post.run(u0, variances=True, copy_back=False)
st = post.kernel_stats()
for pre in ["solve.forward", "solve.forward_off", "solve.backward", "solve.backward_off",
            "selinv.gemm_dmma", "selinv.trsm", "selinv.diag", "selinv.gather", "selinv.mirror"]:
    rows = sorted((int(k.split("@")[1]), v) for k, v in st.items() if k.startswith(pre + "@"))
    tot = sum(v["ms"] for _, v in rows)
    print(pre, "total ms %.2f" % tot)
    for l, v in rows:
        per = v["ms"] / max(v["launches"], 1) * 1e3
        bw = v["bytes"] / (v["ms"] * 1e-3) / 1e9 if v["bytes"] else 0
        fl = v["flops"] / (v["ms"] * 1e-3) / 1e12 if v["flops"] else 0
        print("   lvl %3d  %8.1f us/launch  n=%d  %.0f GB/s  %.2f TF/s  MB=%.1f" %
              (l, per, v["launches"], bw, fl, v["bytes"] / max(v["launches"], 1) / 1e6))
