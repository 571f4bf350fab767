"""Per chunk-level breakdown of one GN-Laplace step's factorizations (GPU)."""
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
cls = ["factor.small_front", "factor.extend_add", "factor.potrf_trsm", "factor.gemm_dmma"]
lv = {}
for k, v in st.items():
    if "@" not in k:
        continue
    name, l = k.split("@")
    if name in cls:
        lv.setdefault(int(l), {})[name] = (v["ms"], v["launches"], (v["flops"] / v["ms"] / 1e9) if v["flops"] else (v["bytes"] / v["ms"] / 1e6))
tot = {c: 0.0 for c in cls}
print("level " + " ".join("%22s" % c.split(".")[1] for c in cls))
for l in sorted(lv):
    row = []
    for c in cls:
        ms, n, a = lv[l].get(c, (0.0, 0, 0.0))
        tot[c] += ms
        row.append("%9.3f/%3d %8.2f" % (ms, n, a))
    print("%5d " % l + " ".join(row))
print({c: round(t, 2) for c, t in tot.items()})
