"""Per chunk-level breakdown of the selected inversion (GPU)."""
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
cls = ["selinv.gather", "selinv.gemm_dmma", "selinv.trsm", "selinv.diag", "selinv.mirror"]
lv = {}
for k, v in st.items():
    if "@" in k and k.split("@")[0] in cls:
        name, l = k.split("@")
        lv.setdefault(int(l), {})[name] = (v["ms"], v["launches"])
tot = {c: 0.0 for c in cls}
print("level " + " ".join("%16s" % c.split(".")[1] for c in cls))
for l in sorted(lv):
    row = []
    for c in cls:
        ms, n = lv[l].get(c, (0.0, 0))
        tot[c] += ms
        row.append("%10.3f/%3d" % (ms, n))
    print("%5d " % l + " ".join(row))
print({c: round(t, 2) for c, t in tot.items()})
