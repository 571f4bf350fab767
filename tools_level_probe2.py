import sys, re
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
for pre in ["solve.forward", "solve.forward_off", "solve.backward", "solve.backward_off"]:
    rows = sorted((int(k.split("@")[1]), v["ms"], v["launches"]) for k, v in st.items() if k.startswith(pre + "@"))
    print(pre, "total ms", round(sum(r[1] for r in rows), 2), [(l, round(ms, 3), n) for l, ms, n in rows])
print({k: round(v["ms"], 2) for k, v in st.items() if "@" not in k})
