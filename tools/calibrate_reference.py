"""Calibrates bench.py's extrapolated reference time for config 4 against the
reference's own MEASURED runs (tests/golden/make_golden_full.py fixtures carry
their stage timings): the 150x150 sample model (bench.reference_sample) is
re-targeted to each measured size with that size's AMD symbolic (flops Σc²,
nnz(L)) and compared with the measured wall time. Output: JSON on stdout
(profiles/r02_reference_calibration.json)."""
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Ref  # noqa: E402


def amd_stats(ref, n_el, n_t):
    p = [1, n_el, -1.0, 1.0, n_t, 1.0, 0.01 / math.pi, 0.5, 10, 1, 1, 10, 2, 1, 1.0, 1e-10, 1e8,
         0, 1e12, 0, 0, 0]
    q = ref.build("spatiotemporal", p).mat("Q_cond")
    perm = ref.amd_order(q.nrows, q.col_ptr, q.row_idx)
    parent, cpl = ref.symbolic(q.nrows, q.col_ptr, q.row_idx, perm)
    c = np.diff(np.asarray(cpl, np.int64)).astype(np.float64)
    return dict(n=q.nrows, nnz_l=float(c.sum()), flops=float((c * c).sum()))


def main():
    import bench
    ref = Ref()
    t0 = time.time()
    sample = bench.reference_sample()  # 150 x 150 measured here, extrapolated to full C4
    out = {"sample": sample["sample"], "sample_stages_s": sample["stages_sample_s"],
           "sample_measured_s": sample["measured_sample_s"], "targets": {}}
    st = sample["stages_sample_s"]
    nfk = [k for k in st if k.startswith("numeric_x")][0]
    # the sample's own AMD stats (same recipe as the targets)
    s0 = amd_stats(ref, *bench.SAMPLE)
    for name, (n_el, n_t) in {"c4_burgers_500.npz": (499, 500),
                              "c4_burgers_full.npz": (999, 1000)}.items():
        path = os.path.join(ROOT, "tests", "golden", name)
        s1 = amd_stats(ref, n_el, n_t)
        sf, sl, sn = s1["flops"] / s0["flops"], s1["nnz_l"] / s0["nnz_l"], s1["n"] / s0["n"]
        pred = (st[nfk] + st["takahashi"]) * sf + st["amd_symbolic"] * sl + st["rest"] * sn
        rec = {"n": s1["n"], "amd_flops": s1["flops"], "amd_nnz_l": s1["nnz_l"],
               "predicted_s": pred}
        if os.path.exists(path):
            times = json.loads(str(np.load(path)["ref_times_json"]))
            rec["measured_s"] = times["t_wall"]
            rec["measured_stages_s"] = times
            rec["model_error"] = pred / times["t_wall"] - 1.0
        out["targets"][name] = rec
    out["wall_s"] = time.time() - t0
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
