"""Partitioned (multi-GPU) factorization, host side: supernode
ownership along the top nested-dissection separators, the cross-edge exchange
schedule, and the torch.distributed transport over gloo with world_size 2
(the same Exchange code NCCL drives on the B200s, here on host buffers).
No GPU needed: the symbolic analysis and the schedule are host code."""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2503_08343_b200 as g
from paper_2503_08343_b200 import partition as pt


def grid_q(nx, ny, shift=0.05):
    k1 = sp.diags([-1.0, 2.0 + shift, -1.0], [-1, 0, 1], (nx, nx))
    k2 = sp.diags([-1.0, 2.0 + shift, -1.0], [-1, 0, 1], (ny, ny))
    k = (sp.kron(sp.eye(ny), k1) + sp.kron(k2, sp.eye(nx))).tocsc()
    q = (k.T @ k + 1e-3 * sp.eye(nx * ny)).tocsc()
    q.sort_indices()
    return g.SparseMatrixCSC.from_scipy(q)


def supernodes(sym):
    ns = int(sym.info.n_supernodes)
    first = np.empty(ns + 1, np.int32)
    rows = np.empty(ns, np.int32)
    level = np.empty(ns, np.int32)
    parent = np.empty(ns, np.int32)
    from paper_2503_08343_b200._capi import i32p, load, ptr
    load().gmrf_symbolic_supernodes(sym._h, ptr(first, i32p), ptr(rows, i32p), ptr(level, i32p),
                                    ptr(parent, i32p))
    return first, rows, level, parent


@pytest.fixture(scope="module")
def sym(lib_built):
    return g.symbolic_analyze(grid_q(48, 40))


@pytest.mark.parametrize("nranks", [1, 2, 4, 8])
def test_owners_are_subtrees(sym, nranks):
    first, rows, level, parent = supernodes(sym)
    o = pt.partition_owners(sym, nranks)
    assert o.min() >= 0 and o.max() < nranks
    if nranks == 1:
        assert not o.any()
        return
    assert len(set(o.tolist())) == nranks  # every rank gets work
    # subtree-to-subcube: every subtree's owners form a contiguous rank range
    # containing its root's owner (ranks only split downwards; a separator sits
    # on the least-loaded rank of the range below it)
    owners = [{int(o[k])} for k in range(len(o))]
    for k in range(len(o)):  # children precede parents
        if parent[k] >= 0:
            owners[parent[k]] |= owners[k]
    for k in range(len(o)):
        lo, hi = min(owners[k]), max(owners[k])
        assert owners[k] == set(range(lo, hi + 1))
        assert lo <= o[k] <= hi
    # balance: the per-rank panel work is within a factor of the mean
    w = np.diff(first)
    work = np.array([sum((r - j) ** 2 for j in range(wk)) for r, wk in zip(rows, w)], float)
    per = np.bincount(o, weights=work, minlength=nranks)
    assert per.min() > 0.15 * per.mean()


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_schedule_is_consistent(sym, nranks):
    first, rows, level, parent = supernodes(sym)
    o = pt.partition_owners(sym, nranks)
    s = pt.partition_schedule(sym, o)
    cross = [k for k in range(len(o)) if parent[k] >= 0 and o[k] != o[parent[k]]]
    assert len(s) == 4 * len(cross)
    w = np.diff(first)
    for phase in range(4):
        ph = s[s[:, 0] == phase]
        assert sorted(ph[:, 4].tolist()) == sorted(cross)
        # ordered by (point, child)
        key = ph[:, 1] * (1 << 32) + ph[:, 4]
        assert np.all(np.diff(key) > 0)
        for _, point, src, dst, c, count in ph:
            p = parent[c]
            r = rows[c] - w[c]
            if phase in (0, 1):  # child → parent
                assert (src, dst) == (o[c], o[p])
            else:  # parent → child
                assert (src, dst) == (o[p], o[c])
            assert count == (r * r if phase in (0, 3) else r)
        if phase == 1:
            assert np.all(ph[:, 1] == level[ph[:, 4]])
        if phase == 2:
            assert np.all(ph[:, 1] == level[parent[ph[:, 4]]])


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _gloo_worker(rank, world, port, q_parts, out):
    """One rank: the C-ABI schedule for a 2-rank partition, then every exchange
    point replayed through TorchExchange(device=False) on host buffers."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q = g.SparseMatrixCSC.from_arrays(*q_parts)
        sym = g.symbolic_analyze(q)
        o = pt.partition_owners(sym, world)
        sched = pt.partition_schedule(sym, o)
        ex = pt.TorchExchange(device=False)
        nr = 3  # right-hand sides for the solve phases
        ok = True
        keep = []
        points = 0
        for phase in range(4):
            ph = sched[sched[:, 0] == phase]
            for point in np.unique(ph[:, 1]):
                msgs, checks = [], []
                for _, _, src, dst, c, count in ph[ph[:, 1] == point]:
                    if rank not in (src, dst):
                        continue
                    cnt = int(count) * (nr if phase in (1, 2) else 1)
                    payload = np.arange(cnt, dtype=np.float64) + 1000.0 * c + 0.25 * phase
                    if src == rank:
                        buf = payload.copy()
                        msgs.append((pt.MSG_SEND, int(dst), int(c), phase, buf.ctypes.data, cnt))
                    else:
                        buf = np.full(cnt, np.nan)
                        msgs.append((pt.MSG_RECV, int(src), int(c), phase, buf.ctypes.data, cnt))
                        checks.append((buf, payload))
                    keep.append(buf)
                if msgs:
                    ex.run(msgs, 0)
                    points += 1
                for buf, payload in checks:
                    ok &= bool(np.array_equal(buf, payload))
        # all-reduces: disjoint column ownership summed exactly; status minimum
        v = np.where(np.arange(10) % world == rank, np.arange(10.0) + 0.5, 0.0)
        st = np.array([7 + rank], np.int32)
        ex.run([(pt.MSG_ALLREDUCE_SUM_F64, -1, -1, -1, v.ctypes.data, 10),
                (pt.MSG_ALLREDUCE_MIN_I32, -1, -1, -1, st.ctypes.data, 1)], 0)
        ok &= bool(np.array_equal(v, np.arange(10.0) + 0.5)) and int(st[0]) == 7
        out[rank] = (ok, len(sched), points)
    finally:
        dist.destroy_process_group()


def test_gloo_exchange_world2(lib_built):
    import torch.multiprocessing as mp
    q = grid_q(32, 30)
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gloo_worker, args=(2, port, (q.nrows, q.ncols, q.col_ptr, q.row_idx, q.values), out),
             nprocs=2, join=True)
    assert out[0][0] and out[1][0], dict(out)
    assert out[0][1] == out[1][1] > 0
    assert out[0][2] > 1 and out[1][2] > 1


# ---- per-rank memory plan (host only) ---------------------------------------
def test_memory_plan_conserves_panels_and_shrinks_per_rank(lib_built):
    """gmrf_partition_memory on the config-5 pipeline's own symbolic (32²×64
    nodes·slices): the ranks' L panels partition the single-GPU panels exactly,
    and every rank needs less memory than one GPU holding the whole factor."""
    import ctypes as C
    from paper_2503_08343_b200 import _capi
    from paper_2503_08343_b200.core import _check
    from paper_2503_08343_b200.spacetime import SpaceTimeSpec, _config
    lib = _capi.load()
    h = C.c_void_p()
    _check(lib.gmrf_spacetime_symbolic(C.byref(_config(SpaceTimeSpec.allen_cahn(31, 64))),
                                       C.byref(h)))
    try:
        one = pt.memory_plan(h, 1)[0]
        info = _capi.SymbolicInfo()
        _check(lib.gmrf_symbolic_info(h, C.byref(info)))
        # panels hold rows × w per supernode: the padded lower trapezoid + the diagonal
        # block's upper triangle
        assert one["l_panels"] >= 8 * info.nnz_l_padded
        for nr in (2, 4, 8):
            plan = pt.memory_plan(h, nr)
            assert sum(p["l_panels"] for p in plan) == one["l_panels"]
            assert sum(p["supernodes"] for p in plan) == info.n_supernodes
            assert max(p["total"] for p in plan) < one["total"]
            assert all(p["u_arena_factor"] <= one["u_arena_factor"] + 8 * info.max_front ** 2
                       for p in plan)
    finally:
        lib.gmrf_symbolic_free(h)


def test_full_config5_memory_plan_fits_four_and_eight_b200s():
    """The committed plan of the full config 5 (128²×256, n = 4.19M;
    tools/memory_plan.py, profiles/r02_c5_memory_plan.json — minutes of host
    symbolic analysis, so generated once; in-place selected inversion,
    load-balanced separator owners): one B200 (180 GB) cannot hold the factor
    (573 GB), 4 ranks fit in HBM (174 GB max), 8 ranks with room to spare."""
    import json
    path = os.path.join(os.path.dirname(__file__), "..", "profiles", "r02_c5_memory_plan.json")
    if not os.path.exists(path):
        pytest.skip("profiles/r02_c5_memory_plan.json not generated")
    plan = json.load(open(path))
    assert plan["n"] == 128 * 128 * 256
    assert plan["ranks"]["1"]["max_total_gb"] > 180.0
    assert plan["ranks"]["4"]["max_total_gb"] < 180.0
    assert plan["ranks"]["8"]["max_total_gb"] < 120.0
