"""Per-level kernel-class times of one config-4 posterior (profiled, serialized):
python tools/phase_levels.py [prefix ...]   (default prefixes: selinv solve)"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402

from paper_2503_08343_b200 import _capi  # noqa: E402
from paper_2503_08343_b200.spacetime import GaussNewtonConfig, SpaceTimePosterior, SpaceTimeSpec  # noqa: E402

prefixes = sys.argv[1:] or ["selinv", "solve"]
spec = SpaceTimeSpec.burgers()
post = SpaceTimePosterior(spec, GaussNewtonConfig(max_iters=1))
u0 = -np.sin(np.pi * spec.node_x())
post.run(u0, variances=True, copy_back=False)
_capi.load().gmrf_spacetime_set_profile(post._h, 2)
post.run(u0, variances=True, copy_back=False)
st = post.kernel_stats()
by = collections.defaultdict(dict)
for name, v in st.items():
    if "@" not in name:
        continue
    base, lvl = name.split("@")
    if any(base.startswith(p) for p in prefixes):
        by[base][int(lvl)] = v
for base in sorted(by):
    tot = sum(v["ms"] for v in by[base].values())
    n = sum(v["launches"] for v in by[base].values())
    print("== %s: %.2f ms, %d launches" % (base, tot, n))
    for lvl in sorted(by[base], reverse=True):
        v = by[base][lvl]
        print("  lvl %3d  %8.1f us  x%d  %s" % (lvl, v["ms"] * 1e3, v["launches"],
              ("%.2f TF/s" % (v["flops"] / v["ms"] / 1e9)) if v["flops"] else (("%.0f GB/s" % (v["bytes"] / v["ms"] / 1e6)) if v["bytes"] else "")))
