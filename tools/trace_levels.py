"""Per-level timeline of one config-4 (or config-5-shape) numeric factorization.

Runs the posterior with GMRF_TRACE set (k_mark markers inside the replayed
graph, factor.cu) and prints, per chunk level, when each launch class started
and ended relative to the factorization's first marker, plus the level's task
counts. Diagnostic only.

usage: python tools/trace_levels.py [c4|c5] [out.txt]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
which = sys.argv[1] if len(sys.argv) > 1 else "c4"
out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "trace_%s.txt" % which)
raw = out + ".raw"
if os.path.exists(raw):
    os.remove(raw)
os.environ["GMRF_TRACE"] = raw

import numpy as np  # noqa: E402

from paper_2503_08343_b200.spacetime import GaussNewtonConfig, SpaceTimePosterior, SpaceTimeSpec  # noqa: E402

if which == "c4":
    spec = SpaceTimeSpec.burgers()
    post = SpaceTimePosterior(spec, GaussNewtonConfig(max_iters=2))
    u0 = -np.sin(np.pi * spec.node_x())
else:
    spec = SpaceTimeSpec.allen_cahn(64, 128)
    post = SpaceTimePosterior(spec, GaussNewtonConfig(max_iters=1))
    u0 = np.random.default_rng(1005).uniform(-0.1, 0.1, spec.n_space)
post.run(u0, variances=False, copy_back=False)
post.run(u0, variances=False, copy_back=False)

blocks, cur = [], []
for line in open(raw):
    if line.startswith("end"):
        blocks.append(cur)
        cur = []
    else:
        cur.append(line)
last = blocks[-1]
rows = []
for line in last:
    a, b = line.split("|")
    t = [int(x) for x in a.split()]
    rows.append((t[0], t[1:], [int(x) for x in b.split()]))
t0 = min(min(x for x in r[1] if x) for r in rows)
names = "lvl  ea_s   ea_e/pan_s pan_e  gm_s  gm_e | rest_s rest_e | uu_s uu_e | nsm ean chunks slabs trsm gmn grn onewave"
with open(out, "w") as f:
    f.write("# us since the first marker; slots: 8 ea start, 0 ea end, 1 panel end, 2 next-GEMM start, 3 next-GEMM end, 4/5 bulk start/end\n")
    f.write(names + "\n")
    prev_end = 0.0
    for lvl, t, c in rows:
        u = [(x - t0) / 1e3 if x else -1 for x in t]
        f.write("%3d %8.1f %8.1f %8.1f %8.1f %8.1f | %8.1f %8.1f | %s | ea %.1f pan %.1f gm %.1f rest %.1f\n" % (
            lvl, u[8], u[0], u[1], u[2], u[3], u[4], u[5], " ".join(map(str, c)),
            u[0] - u[8], u[1] - u[0], u[3] - u[2], u[5] - u[4]))
    f.write("total %.1f us\n" % ((max(max(r[1]) for r in rows) - t0) / 1e3))
print(open(out).read()[-3000:])
