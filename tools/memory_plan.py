"""Per-rank device-memory plan of the ND-partitioned config-5 posterior from the
host symbolic alone (no GPU): python tools/memory_plan.py [n_cells n_t] > plan.json

Builds the pipeline's master pattern and geometric nested dissection
(gmrf_spacetime_symbolic), partitions the supernodal tree for 1/2/4/8 ranks
(subtree-to-subcube, gmrf_partition_owners) and sizes every rank's L panels,
Σ panels, lifetime-packed update-matrix arenas and replicated pattern data
(gmrf_partition_memory)."""
import ctypes as C
import json
import os
import resource
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2503_08343_b200 import _capi  # noqa: E402
from paper_2503_08343_b200.core import _check  # noqa: E402
from paper_2503_08343_b200.partition import memory_plan  # noqa: E402
from paper_2503_08343_b200.spacetime import SpaceTimeSpec, _config  # noqa: E402


def main():
    n_cells, n_t = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (127, 256)
    spec = SpaceTimeSpec.allen_cahn(n_cells=n_cells, n_t=n_t)
    lib = _capi.load()
    t0 = time.time()
    h = C.c_void_p()
    _check(lib.gmrf_spacetime_symbolic(C.byref(_config(spec)), C.byref(h)))
    t_sym = time.time() - t0
    info = _capi.SymbolicInfo()
    _check(lib.gmrf_symbolic_info(h, C.byref(info)))
    out = {"workload": f"config 5: Allen-Cahn space-time GMRF, {n_cells + 1}^2 nodes x {n_t} slices",
           "n": info.n, "nnz_pattern": info.nnz_q, "nnz_l": info.nnz_l,
           "nnz_l_padded": info.nnz_l_padded, "flops_per_factorization": info.flops_ref,
           "supernodes": info.n_supernodes, "max_front": info.max_front,
           "host_symbolic_s": t_sym, "b200_hbm_gb": 180.0, "ranks": {}}
    for nr in (1, 2, 4, 8):
        plan = memory_plan(h, nr)
        out["ranks"][str(nr)] = {
            "max_total_gb": max(p["total"] for p in plan) / 1e9,
            "per_rank_gb": [{k: (v / 1e9 if k != "supernodes" else v) for k, v in p.items()}
                            for p in plan]}
    lib.gmrf_symbolic_free(h)
    out["host_peak_rss_gb"] = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
