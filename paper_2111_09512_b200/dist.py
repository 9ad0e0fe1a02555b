"""Multi-GPU view of the C ABI (ilug_dist_*): row-block partition, halo plans
and the NCCL-backed block-Jacobi ILU smoother, one process per GPU.

torch.distributed (gloo or nccl) is only plumbing here: it moves the 128-byte
NCCL id and the halo request lists between ranks at setup. The data path
(halo exchange, sweeps) is NCCL + libilug kernels.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, List

import numpy as np

from . import Config, IlugError, Matrix, _as, _check, _host_ptrs, _ptr, _stream, lib


def _prefer_torch_nccl() -> None:
    """libilug binds NCCL lazily (dlopen). Point it at torch's bundled NCCL so a
    process that imports torch (before or after) ends up with one NCCL copy."""
    import os
    if os.environ.get("ILUG_NCCL_LIB"):
        return
    try:
        import nvidia.nccl as nn  # torch's pip dependency
        for base in list(getattr(nn, "__path__", [])):
            cand = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["ILUG_NCCL_LIB"] = cand
                return
    except ImportError:
        pass


_prefer_torch_nccl()


def partition(n: int, nranks: int) -> np.ndarray:
    starts = np.empty(nranks + 1, np.int64)
    _check(lib.ilug_dist_partition(n, nranks, _as(starts, C.c_longlong)))
    return starts


def generate_rows(spec: str, row0: int, row1: int) -> Matrix:
    out = C.c_void_p()
    _check(lib.ilug_dist_generate_rows(spec.encode(), row0, row1, C.byref(out)))
    return Matrix(out.value)


class Plan:
    """Halo plan of one rank's rows (global column ids)."""

    def __init__(self, rows: Matrix, n_global: int, nranks: int, rank: int):
        out = C.c_void_p()
        _check(lib.ilug_dist_plan_create(rows.h, n_global, nranks, rank, C.byref(out)))
        self._init(out, nranks, rank)

    def _init(self, h, nranks, rank):
        self.h = h
        self.nranks, self.rank = nranks, rank
        r0, r1, nh = C.c_longlong(), C.c_longlong(), C.c_longlong()
        _check(lib.ilug_dist_plan_info(self.h, C.byref(r0), C.byref(r1), C.byref(nh)))
        self.row0, self.row1, self.nhalo = r0.value, r1.value, nh.value

    @classmethod
    def _adopt(cls, h, nranks, rank) -> "Plan":
        p = cls.__new__(cls)
        p._init(h, nranks, rank)
        return p

    def exchange(self, comm: "Comm") -> None:
        """Complete the send lists over the communicator (collective)."""
        _check(lib.ilug_dist_plan_exchange(self.h, comm.h))

    def requests(self, q: int) -> np.ndarray:
        cnt = lib.ilug_dist_plan_requests(self.h, q, None)
        ids = np.empty(max(cnt, 0), np.int64)
        if cnt > 0:
            lib.ilug_dist_plan_requests(self.h, q, _as(ids, C.c_longlong))
        return ids

    def set_sends(self, q: int, ids) -> None:
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        _check(lib.ilug_dist_plan_set_sends(self.h, q, _as(ids, C.c_longlong), len(ids)))

    def sends(self, q: int) -> np.ndarray:
        cnt = lib.ilug_dist_plan_sends(self.h, q, None)
        rows = np.empty(max(cnt, 0), np.int64)
        if cnt > 0:
            lib.ilug_dist_plan_sends(self.h, q, _as(rows, C.c_longlong))
        return rows

    def matrix(self, which: str = "ext") -> Matrix:
        out = C.c_void_p()
        _check(lib.ilug_dist_plan_matrix(self.h, {"ext": 0, "diag": 1, "off": 2}[which], C.byref(out)))
        return Matrix(out.value)

    def exchange_requests(self, all_gather: Callable[[object], List[object]]) -> None:
        """Tell every rank what we need from it; record what it needs from us.
        all_gather(obj) -> list over ranks (e.g. torch.distributed.all_gather_object)."""
        mine = {q: self.requests(q).tolist() for q in range(self.nranks) if q != self.rank}
        everyone = all_gather(mine)
        for q in range(self.nranks):
            if q != self.rank:
                wanted = everyone[q].get(self.rank, [])
                if wanted:
                    self.set_sends(q, wanted)

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and lib is not None:
            lib.ilug_dist_plan_free(self.h)
            self.h = C.c_void_p()


def unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib.ilug_dist_unique_id(C.cast(buf, C.c_void_p)))
    return buf.raw


class Comm:
    """One rank's communicator: NCCL (one process per GPU) or an in-process
    rank group (``LocalGroup``: threads of one process, several may share a GPU)."""

    def __init__(self, nranks: int, rank: int, uid: bytes = None, group: "LocalGroup" = None):
        out = C.c_void_p()
        if group is not None:
            _check(lib.ilug_dist_comm_create_local(group.h, rank, C.byref(out)))
            self.group = group  # keep the group alive
        else:
            buf = C.create_string_buffer(uid, 128)
            _check(lib.ilug_dist_comm_create(nranks, rank, C.cast(buf, C.c_void_p), C.byref(out)))
        self.h = out
        self.nranks, self.rank = nranks, rank

    def allreduce_sum(self, t, count: int, stream=None) -> None:
        _check(lib.ilug_dist_allreduce_sum(self.h, _ptr(t, count), count, _stream(stream)))

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and lib is not None:
            lib.ilug_dist_comm_free(self.h)
            self.h = C.c_void_p()


class LocalGroup:
    """In-process rank group (ilug_dist_group): ranks are host threads; every
    collective synchronises the caller's stream and meets at a host barrier."""

    def __init__(self, nranks: int):
        out = C.c_void_p()
        _check(lib.ilug_dist_group_create(nranks, C.byref(out)))
        self.h = out
        self.nranks = nranks

    def comm(self, rank: int) -> Comm:
        return Comm(self.nranks, rank, group=self)

    def abort(self) -> None:
        """Release the other ranks of a failed collective (their calls raise)."""
        lib.ilug_dist_group_abort(self.h)

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and lib is not None:
            lib.ilug_dist_group_free(self.h)
            self.h = C.c_void_p()


def run_ranks(nranks: int, fn: Callable[[int], object], group: "LocalGroup" = None) -> List[object]:
    """fn(rank) on nranks host threads (ctypes drops the GIL inside the C ABI,
    so the ranks' collectives meet); the first exception aborts the group
    (the other ranks' pending collectives fail instead of waiting) and is re-raised."""
    import threading
    out: List[object] = [None] * nranks
    err: List[BaseException] = []

    def body(r):
        try:
            import torch
            torch.cuda.set_device(0)
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            err.append(e)
            if group is not None:
                group.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return out


class Smoother:
    """Rank-local smoother of a distributed matrix (global residual): block-Jacobi
    ILU / poly-GS, hybrid Gauss-Seidel, Jacobi / l1-Jacobi."""

    def __init__(self, plan: Plan, comm: Comm, cfg: Config):
        out = C.c_void_p()
        _check(lib.ilug_dist_smoother_create(plan.h, comm.h, cfg.h, C.byref(out)))
        self.h = out
        self.n = plan.row1 - plan.row0

    def smooth(self, b, x, stream=None):
        _check(lib.ilug_dist_smooth(self.h, _ptr(b, self.n), _ptr(x, self.n), _stream(stream)))

    def residual(self, x, b, r, stream=None):
        _check(lib.ilug_dist_residual(self.h, _ptr(x, self.n), _ptr(b, self.n), _ptr(r, self.n), _stream(stream)))

    def smooth_host_many(self, bs, xs):
        """Pipelined host-buffer smoothing (ilug_dist_smooth_host_many); collective."""
        _check(lib.ilug_dist_smooth_host_many(self.h, len(bs), _host_ptrs(bs, self.n), _host_ptrs(xs, self.n)))

    def stats(self):
        v = [C.c_longlong() for _ in range(4)]
        _check(lib.ilug_dist_smoother_stats(self.h, *[C.byref(x) for x in v]))
        return dict(zip(("nloc", "nnz_A", "nnz_Ls", "nnz_Us"), (x.value for x in v)))

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and lib is not None:
            lib.ilug_dist_smoother_free(self.h)
            self.h = C.c_void_p()


class Solver:
    """Distributed GMRES+AMG over a row-block partition of the GLOBAL hierarchy
    (every rank passes the same host hierarchy): halo-exchanged A/R/P products,
    rank-local smoothers, replicated coarsest solve, summed GMRES reductions."""

    def __init__(self, hierarchy, comm: Comm):
        out = C.c_void_p()
        _check(lib.ilug_dist_solver_create(hierarchy.h, comm.h, C.byref(out)))
        self.h = out
        r0, nl, lv = C.c_longlong(), C.c_longlong(), C.c_int()
        _check(lib.ilug_dist_solver_info(self.h, C.byref(r0), C.byref(nl), C.byref(lv)))
        self.row0, self.nloc, self.levels = r0.value, nl.value, lv.value

    def vcycle(self, r, z, stream=None):
        _check(lib.ilug_dist_vcycle(self.h, _ptr(r, self.nloc), _ptr(z, self.nloc), _stream(stream)))

    def gmres(self, cfg: Config, b, x, stream=None):
        it, rr = C.c_longlong(), C.c_double()
        st = lib.ilug_dist_gmres(self.h, cfg.h, _ptr(b, self.nloc), _ptr(x, self.nloc), C.byref(it), C.byref(rr),
                                 _stream(stream))
        _check(st, allow_not_converged=True)
        return dict(status=st, iterations=it.value, final_relres=rr.value)

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and lib is not None:
            lib.ilug_dist_solver_free(self.h)
            self.h = C.c_void_p()


class LevelPlans:
    """Host-only per-level distribution of a hierarchy for one rank
    (ilug_dist_level_plans): the halo plans the distributed V-cycle uses."""

    def __init__(self, hierarchy, nranks: int, rank: int):
        out = C.c_void_p()
        _check(lib.ilug_dist_level_plans(hierarchy.h, nranks, rank, C.byref(out)))
        self.h = out
        self.nranks, self.rank = nranks, rank
        self.count = lib.ilug_dist_levels_count(self.h)

    def plan(self, k: int, which: str = "A") -> Plan:
        out = C.c_void_p()
        _check(lib.ilug_dist_levels_plan(self.h, k, {"A": 0, "R": 1, "P": 2}[which], C.byref(out)))
        return Plan._adopt(out, self.nranks, self.rank)

    def last(self, which: str) -> Matrix:
        out = C.c_void_p()
        _check(lib.ilug_dist_levels_last(self.h, {"R": 0, "P": 1}[which], C.byref(out)))
        return Matrix(out.value)

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and lib is not None:
            lib.ilug_dist_levels_free(self.h)
            self.h = C.c_void_p()


__all__ = ["partition", "generate_rows", "Plan", "unique_id", "Comm", "LocalGroup", "run_ranks", "Smoother",
           "Solver", "LevelPlans", "IlugError"]
