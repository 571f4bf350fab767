import sys, json, re
import numpy as np
sys.path.insert(0, '.')
from paper_2503_08343_b200.spacetime import SpaceTimePosterior, SpaceTimeSpec, GaussNewtonConfig
spec = SpaceTimeSpec.burgers()
post = SpaceTimePosterior(spec, GaussNewtonConfig(max_iters=1))
u0 = -np.sin(np.pi * spec.node_x())
post.run(u0, variances=False, copy_back=False)
post.set_profile(2)
post.run(u0, variances=False, copy_back=False)
st = post.kernel_stats()
rows = {}
for k, v in st.items():
    m = re.match(r"(.*)@(\d+)$", k)
    if m:
        rows.setdefault(int(m.group(2)), {})[m.group(1)] = (v["ms"], v["launches"], v["flops"], v["bytes"])
for l in sorted(rows):
    print(l, {k: (round(a[0], 3), a[1], "%.2e" % a[2]) for k, a in rows[l].items()})
print({k: round(v["ms"], 2) for k, v in st.items() if "@" not in k})
