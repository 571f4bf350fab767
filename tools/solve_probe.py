"""Per supernode-level breakdown of the config-4 solves (profiled, serialized):
ms, algorithmic bytes and GB/s per level for solve.* kernel classes."""
import re
import sys
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
    m = re.match(r"(solve\..*)@(\d+)$", k)
    if m:
        rows.setdefault(int(m.group(2)), {})[m.group(1)] = v
tb = tt = 0.0
for l in sorted(rows):
    out = []
    for k, v in sorted(rows[l].items()):
        out.append("%s %.3f ms %d x %.1f MB %.0f GB/s" % (k, v["ms"], v["launches"], v["bytes"] / 1e6,
                                                      v["bytes"] / max(v["ms"], 1e-9) / 1e6))
        tb += v["bytes"]
        tt += v["ms"]
    print(l, " | ".join(out))
print("total %.3f ms %.1f MB %.0f GB/s" % (tt, tb / 1e6, tb / tt / 1e6))
