"""Partitioned (multi-GPU) factorization — SURVEY §8(e).

The supernodal elimination tree is split along its top nested-dissection
separators (``gmrf_partition_owners``: subtree-to-subcube, whole subtrees per
rank, each separator on the lowest rank of the range below it). Each rank
stores and factors its own supernodes on its GPU; the data that crosses ranks
moves at fixed exchange points (``include/gmrf_b200.h``, gmrf_msg_t):

* factorization: the update matrix (Schur-complement contribution) of a child
  goes to its parent's rank before the parent's extend-add;
* forward solve: the child's update vector, the same way;
* backward solve: x on the child's below-diagonal rows, parent → child;
* selected inversion: Σ on those rows, parent → child;
* results (status, x, variances) are all-reduced, so every rank returns the
  complete answer — the reference API semantics are unchanged.

The library calls back into an ``Exchange`` here for the transport:

* ``TorchExchange`` — torch.distributed point-to-point + all-reduce. On GPUs
  (backend ``nccl``) the messages are device buffers enqueued on the factor's
  stream: NVLink/NVSwitch between the B200s of one box. On CPU (``gloo``) the
  same code moves host buffers (tests).
* ``NcclExchange`` — the native transport: ``ncclSend`` / ``ncclRecv`` /
  ``ncclAllReduce`` posted by the library itself on the factor's stream
  (csrc/nccl_exchange.cpp), no Python at the exchange points.
* ``LoopbackGroup`` — several ranks in one process on one GPU (tests): each
  rank runs in its own thread, messages are device-to-device copies matched by
  (src, dst, phase, child). Host-side waits only; no kernel waits on another
  rank's kernel.

The reference is single-threaded and has no distributed
path; this module has no reference counterpart beyond the API it keeps
(cholesky.hpp:164-227, takahashi.hpp:67).
"""
from __future__ import annotations

import ctypes as C
import threading
import traceback

import numpy as np

from . import _capi
from ._capi import i32p, i64p, ptr
from .core import CholeskyFactor, SymbolicFactor, _check, cholesky_refactor  # noqa: F401

MSG_SEND, MSG_RECV, MSG_ALLREDUCE_SUM_F64, MSG_ALLREDUCE_MIN_I32 = 0, 1, 2, 3
PHASES = {0: "factor", 1: "fsolve", 2: "bsolve", 3: "selinv"}


def partition_owners(sym: SymbolicFactor, nranks: int) -> np.ndarray:
    """Owner rank of every supernode (host only)."""
    o = np.empty(int(sym.info.n_supernodes), np.int32)
    _check(_capi.load().gmrf_partition_owners(sym._h, int(nranks), ptr(o, i32p)))
    return o


def partition_schedule(sym: SymbolicFactor, owner) -> np.ndarray:
    """All cross-edge messages: rows (phase, point, src, dst, child, count)."""
    lib = _capi.load()
    o = np.ascontiguousarray(owner, np.int32)
    n = C.c_int64()
    _check(lib.gmrf_partition_schedule(sym._h, ptr(o, i32p), None, C.byref(n)))
    rows = np.empty((n.value, 6), np.int64)
    _check(lib.gmrf_partition_schedule(sym._h, ptr(o, i32p), ptr(rows, i64p), C.byref(n)))
    return rows


class Exchange:
    """Wraps ``run(msgs, stream)`` as the C exchange callback. ``msgs`` is a list
    of (kind, peer, tag, phase, dptr, count) tuples; ``stream`` the cudaStream_t
    (int) the factor enqueues on. Exceptions are reported and turned into a
    nonzero return, which the library raises as a device error."""

    def __init__(self):
        self.fn = _capi.EXCHANGE_FN(self._cb)
        self.calls = 0
        self.bytes = 0

    def _cb(self, ctx, msgs, count, stream):
        try:
            ms = [(m.kind, m.peer, m.tag, m.phase, m.dptr, m.count)
                  for m in (msgs[i] for i in range(count))]
            self.calls += 1
            self.bytes += sum(8 * m[5] for m in ms if m[0] == MSG_SEND)
            self.run(ms, stream or 0)
            return 0
        except Exception:  # noqa: BLE001 - reported, then surfaced by the library
            traceback.print_exc()
            return 1

    def run(self, msgs, stream):  # pragma: no cover - abstract
        raise NotImplementedError


class _CudaArray:
    """Minimal __cuda_array_interface__ view of a raw device pointer."""

    def __init__(self, p, count, typestr):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                         "data": (int(p), False), "version": 3,
                                         "strides": None, "stream": None}


def _typestr(kind):
    return "<i4" if kind == MSG_ALLREDUCE_MIN_I32 else "<f8"


def device_tensor(p, count, kind=MSG_SEND):
    import torch
    return torch.as_tensor(_CudaArray(p, count, _typestr(kind)), device="cuda")


def host_tensor(p, count, kind=MSG_SEND):
    import torch
    ct = C.c_int32 if kind == MSG_ALLREDUCE_MIN_I32 else C.c_double
    a = np.ctypeslib.as_array(C.cast(C.c_void_p(p), C.POINTER(ct)), shape=(int(count),))
    return torch.from_numpy(a)


class TorchExchange(Exchange):
    """torch.distributed transport. ``device=True``: NCCL on device buffers,
    enqueued on the factor's stream (torch's current stream is set to it, and
    the returned works make it wait for the transfers); ``device=False``: host
    buffers (gloo, CPU tests)."""

    def __init__(self, group=None, device=True):
        super().__init__()
        import torch
        import torch.distributed as dist
        self.group = group
        self.device = device
        if device:
            # NCCL: the first point-to-point batch must not be the group's first
            # collective (torch batch_isend_irecv contract) — warm the communicator
            t = torch.zeros(1, device="cuda")
            dist.all_reduce(t, group=group)
            torch.cuda.synchronize()

    def _tensor(self, p, count, kind):
        return device_tensor(p, count, kind) if self.device else host_tensor(p, count, kind)

    def run(self, msgs, stream):
        import torch
        import torch.distributed as dist

        def body():
            ops = []
            for kind, peer, tag, phase, p, count in msgs:
                if kind in (MSG_SEND, MSG_RECV):
                    t = self._tensor(p, count, kind)
                    ops.append(dist.P2POp(dist.isend if kind == MSG_SEND else dist.irecv, t,
                                          peer, self.group, tag if not self.device else 0))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            for kind, peer, tag, phase, p, count in msgs:
                if kind == MSG_ALLREDUCE_SUM_F64:
                    dist.all_reduce(self._tensor(p, count, kind), op=dist.ReduceOp.SUM,
                                    group=self.group)
                elif kind == MSG_ALLREDUCE_MIN_I32:
                    dist.all_reduce(self._tensor(p, count, kind), op=dist.ReduceOp.MIN,
                                    group=self.group)

        if self.device and stream:
            with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                body()
        else:
            body()


class NcclExchange:
    """Native NCCL transport (csrc/nccl_exchange.cpp): the library posts
    ncclSend / ncclRecv / ncclAllReduce on the factor's stream itself — no Python
    at the exchange points. One communicator per process over ``nranks`` ranks;
    rank 0's unique id is broadcast with torch.distributed (any backend), or pass
    ``unique_id`` (128 bytes) obtained otherwise. The current CUDA device must be
    the one this rank uses."""

    def __init__(self, nranks=None, rank=None, unique_id=None, group=None):
        lib = _capi.load()
        if nranks is None or rank is None:
            import torch.distributed as dist
            nranks, rank = dist.get_world_size(group), dist.get_rank(group)
        if unique_id is None:
            uid = (C.c_uint8 * 128)()
            if rank == 0:
                _check_nccl(lib, lib.gmrf_nccl_unique_id(uid))
            if nranks > 1:
                import torch.distributed as dist
                box = [bytes(uid)]
                dist.broadcast_object_list(box, src=0, group=group)
                uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
        else:
            uid = (C.c_uint8 * 128).from_buffer_copy(bytes(unique_id))
        comm = C.c_void_p()
        _check_nccl(lib, lib.gmrf_nccl_comm_create(int(nranks), int(rank), uid, C.byref(comm)))
        self.ctx = comm
        self.fn = lib.gmrf_nccl_exchange()
        self.nranks, self.rank = int(nranks), int(rank)

    def close(self):
        if getattr(self, "ctx", None):
            _capi.load().gmrf_nccl_comm_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        self.close()


def _check_nccl(lib, rc):
    if rc != 0:
        from .core import DeviceError
        raise DeviceError(lib.gmrf_nccl_last_error().decode() or "NCCL transport failed")


class LoopbackGroup:
    """``nranks`` ranks of a partitioned factor inside one process on one GPU
    (tests): ``exchange(rank)`` gives each rank's transport; run each rank's
    calls in its own thread (``run_ranks``)."""

    def __init__(self, nranks: int, timeout: float = 180.0):
        self.n = nranks
        self.timeout = timeout  # a mismatched schedule fails instead of hanging
        self.cv = threading.Condition()
        self.mail = {}
        self.consumed = set()
        self.barrier = threading.Barrier(nranks, timeout=timeout)
        self.slots = [None] * nranks
        self.result = None

    def exchange(self, rank: int) -> Exchange:
        grp = self

        class _Loop(Exchange):
            def run(self, msgs, stream):
                grp._run(rank, msgs, stream)

        return _Loop()

    def _run(self, rank, msgs, stream):
        import torch
        # this rank's sends are complete (stream 0: the legacy default stream)
        if stream:
            torch.cuda.ExternalStream(stream).synchronize()
        else:
            torch.cuda.synchronize()
        sends = [m for m in msgs if m[0] == MSG_SEND]
        recvs = [m for m in msgs if m[0] == MSG_RECV]
        with self.cv:
            for kind, peer, tag, phase, p, count in sends:
                self.mail[(rank, peer, phase, tag)] = (p, count)
            self.cv.notify_all()
        for kind, peer, tag, phase, p, count in recvs:
            key = (peer, rank, phase, tag)
            with self.cv:
                if not self.cv.wait_for(lambda: key in self.mail, self.timeout):
                    raise TimeoutError(f"loopback rank {rank}: no message {key}")
                sp, sc = self.mail.pop(key)
            if sc != count:
                raise RuntimeError(f"loopback: size mismatch {key}: {sc} != {count}")
            device_tensor(p, count).copy_(device_tensor(sp, count))
            torch.cuda.synchronize()
            with self.cv:
                self.consumed.add(key)
                self.cv.notify_all()
        with self.cv:  # the peers have copied everything this rank sent
            keys = [(rank, peer, phase, tag) for _, peer, tag, phase, _, _ in sends]
            if not self.cv.wait_for(lambda: all(k in self.consumed for k in keys), self.timeout):
                raise TimeoutError(f"loopback rank {rank}: sends not consumed {keys}")
            self.consumed.difference_update(keys)
        for kind, peer, tag, phase, p, count in msgs:
            if kind in (MSG_ALLREDUCE_SUM_F64, MSG_ALLREDUCE_MIN_I32):
                self._allreduce(rank, kind, p, count)

    def _allreduce(self, rank, kind, p, count):
        import torch
        self.slots[rank] = device_tensor(p, count, kind)
        self.barrier.wait()
        if rank == 0:
            acc = self.slots[0].clone()
            for t in self.slots[1:]:
                acc = acc + t if kind == MSG_ALLREDUCE_SUM_F64 else torch.minimum(acc, t)
            self.result = acc
            torch.cuda.synchronize()
        self.barrier.wait()
        self.slots[rank].copy_(self.result)
        torch.cuda.synchronize()
        self.barrier.wait()

    def run_ranks(self, fn):
        """Calls fn(rank) for every rank concurrently; returns the results in rank
        order and re-raises the first exception."""
        out = [None] * self.n
        err = [None] * self.n

        def go(r):
            try:
                out[r] = fn(r)
            except BaseException as e:  # noqa: BLE001
                err[r] = e
                self.barrier.abort()
                with self.cv:
                    self.cv.notify_all()

        ts = [threading.Thread(target=go, args=(r,)) for r in range(self.n)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for e in err:
            if e is not None:
                raise e
        return out


class PartitionedFactor(CholeskyFactor):
    """This rank's share of an ND-partitioned factor. ``refactor``, ``solve``,
    ``solve_triangular`` and ``takahashi_diagonal`` work as on CholeskyFactor and
    return complete results on every rank; ``L`` and the full selected inverse
    are not assembled (the factor is distributed)."""

    def __init__(self, sym: SymbolicFactor, nranks: int, rank: int, exchange: Exchange,
                 owner=None):
        self.sym = sym
        self.nranks, self.rank = int(nranks), int(rank)
        self._exchange = exchange  # keeps the C callback alive
        o = None if owner is None else np.ascontiguousarray(owner, np.int32)
        h = C.c_void_p()
        _check(_capi.load().gmrf_factor_create_partitioned(sym._h, self.nranks, self.rank,
                                                           ptr(o, i32p), exchange.fn,
                                                           getattr(exchange, "ctx", None),
                                                           C.byref(h)))
        self._h = h
        self.perm = sym.perm
        self.perm_inv = sym.perm_inv
        self._L = None


def cholesky_factor_partitioned(q, sym: SymbolicFactor | None = None, group=None, exchange=None):
    """cholesky_factor (cholesky.hpp:164) across the ranks of a torch.distributed
    group: every rank passes the same Q and gets its PartitionedFactor."""
    import torch.distributed as dist
    from .core import symbolic_analyze
    sym = sym or symbolic_analyze(q)
    nranks = dist.get_world_size(group)
    rank = dist.get_rank(group)
    exchange = exchange or TorchExchange(group, device=True)
    f = PartitionedFactor(sym, nranks, rank, exchange)
    f.refactor(q.values)
    return f


MEMORY_FIELDS = ("l_panels", "sigma_panels", "u_arena_factor", "u_arena_selinv", "replicated",
                 "total", "supernodes")


def memory_plan(sym_handle, nranks: int, owner=None):
    """Per-rank device-memory plan (bytes) of a partitioned factorization with
    selected inversion, from a symbolic handle alone (host only):
    gmrf_partition_memory. Returns a list of dicts, one per rank."""
    import ctypes as C
    import numpy as np
    from . import _capi
    from ._capi import i32p, i64p, ptr
    from .core import _check
    rows = np.zeros((nranks, 7), np.int64)
    own = None if owner is None else np.ascontiguousarray(owner, np.int32)
    _check(_capi.load().gmrf_partition_memory(sym_handle, int(nranks), ptr(own, i32p),
                                              ptr(rows, i64p)))
    return [dict(zip(MEMORY_FIELDS, map(int, r))) for r in rows]
