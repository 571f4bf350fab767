"""Perf probe: factor/solve/selinv timings on reference-built problems (uses oracle/_ref)."""
import json, sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_2503_08343_b200 as g
from oracle.pyoracle import Ref
import torch
ref = Ref()
which = sys.argv[1:] or ["c2"]
res = {}
def run(name, Qm):
    q = g.SparseMatrixCSC.from_arrays(Qm.nrows, Qm.ncols, Qm.col_ptr, Qm.row_idx, Qm.values)
    t = time.perf_counter(); sym = g.symbolic_analyze(q); ts = time.perf_counter() - t
    f = g.CholeskyFactor(sym)
    f.refactor(q.values)
    tn = []
    for _ in range(3):
        torch.cuda.synchronize(); t = time.perf_counter(); f.refactor(q.values); tn.append(time.perf_counter() - t)
    b = np.ones(q.nrows)
    tsv = []
    for _ in range(3):
        t = time.perf_counter(); x = g.solve(f, b); tsv.append(time.perf_counter() - t)
    bb = np.ones((q.nrows, 16))
    t = time.perf_counter(); x = g.solve(f, bb); t16 = time.perf_counter() - t
    tv = []
    for _ in range(2):
        t = time.perf_counter(); v = g.takahashi_diagonal(f); tv.append(time.perf_counter() - t)
    i = sym.info; st = f.stats()
    res[name] = dict(n=q.nrows, nnzL=i.nnz_l, nnzLpad=i.nnz_l_padded, ns=i.n_supernodes, lev=i.n_levels,
        maxfront=i.max_front, flops=i.flops_ref, flops_sn=i.flops_sn, U=i.update_entries,
        symbolic_s=ts, numeric_s=min(tn), tflops=i.flops_ref/min(tn)/1e12, solve_s=min(tsv), solve16_s=t16,
        selinv_s=min(tv), launches=[st.launches_numeric, st.launches_solve, st.launches_selinv],
        dev_gb=st.device_bytes/1e9)
    print(name, json.dumps(res[name]), flush=True)
if "c2" in which:
    b = ref.build("matern2d", [255, 10, 2, 1, 2000, 1002, 400, 0.05, 0, 2002, 0]); run("c2", b.mat("Q_post"))
if "c3" in which:
    b = ref.build("spatiotemporal", [0, 499, 0.0, 1.0, 1000, 1.0, 0.1, 0.0, 10, 1, 1, 10, 2, 1, 1.0, 1e-10, 1e6, 1003, 0, 0, 0, 0])
    run("c3", b.mat("Q_cond"))
if "c3s" in which:
    b = ref.build("spatiotemporal", [0, 199, 0.0, 1.0, 400, 1.0, 0.1, 0.0, 10, 1, 1, 10, 2, 1, 1.0, 1e-10, 1e6, 1003, 0, 0, 0, 0])
    run("c3s", b.mat("Q_cond"))
