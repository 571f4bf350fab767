"""Per-level panel time (profiled, serialized) for the config-4 factorization."""
import re, sys
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
    m = re.match(r"(factor\.[a-z_]+)@(\d+)$", k)
    if m:
        rows.setdefault(int(m.group(2)), {})[m.group(1)] = v["ms"] / v["launches"] * 1e3
for l in sorted(rows):
    print(l, " ".join(f"{k.split('.')[1]}={v:.1f}us" for k, v in sorted(rows[l].items())))
