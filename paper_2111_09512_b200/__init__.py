"""B200-native ILU-smoother / AMG / GMRES solve phase (arXiv 2111.09512).

Python view of the C ABI in ``include/iluamg_b200.h`` (the reference's
``iluamg_*`` entry points, include/iluamg.h:36-132) and ``include/ilug.h``
(device handles for each hot-path subsystem). Every compute call goes through
``libilug.so`` (sm_100a kernels + native host setup); there is no Python or
CPU compute path, and importing fails loudly when the library is missing.

Device arrays are passed as anything with ``data_ptr()`` (torch CUDA tensors)
or raw integer pointers; streams as ``torch.cuda.Stream`` / raw handles.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

__all__ = [
    "lib", "IlugError", "Matrix", "Config", "Report", "Factors", "DeviceMatrix",
    "Smoother", "Hierarchy", "run_solve", "run_bench_trisolve", "run_schur_solve",
    "run_analyze", "config_reference", "device_count", "LIB_PATH",
]

OK, NOT_CONVERGED, ERR_INVALID, ERR_NUMERIC = 0, 1, 2, 3
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libilug.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it first (python -c 'import __graft_entry__ as g; g.build()' "
        "or make -C paper_2111_09512_b200/csrc). There is no CPU fallback.")
lib = C.CDLL(LIB_PATH)

_vp, _i, _ll, _d = C.c_void_p, C.c_int, C.c_longlong, C.c_double
_pvp, _pll, _pd, _pi = C.POINTER(C.c_void_p), C.POINTER(C.c_longlong), C.POINTER(C.c_double), C.POINTER(C.c_int)
_cs = C.c_char_p

_SIGS = {
    # iluamg_* drop-in
    "iluamg_version": (_cs, []), "iluamg_last_error": (_cs, []),
    "iluamg_matrix_read": (_i, [_cs, _pvp]), "iluamg_matrix_generate": (_i, [_cs, _pvp]),
    "iluamg_matrix_write": (_i, [_vp, _cs]), "iluamg_matrix_rows": (_ll, [_vp]),
    "iluamg_matrix_cols": (_ll, [_vp]), "iluamg_matrix_nnz": (_ll, [_vp]),
    "iluamg_matrix_free": (None, [_vp]),
    "iluamg_config_create": (_i, [_pvp]), "iluamg_config_load": (_i, [_vp, _cs]),
    "iluamg_config_set": (_i, [_vp, _cs, _cs]), "iluamg_config_get": (_cs, [_vp, _cs]),
    "iluamg_config_reference": (_cs, []), "iluamg_config_free": (None, [_vp]),
    "iluamg_run_analyze": (_i, [_vp, _vp, _pvp]), "iluamg_run_solve": (_i, [_vp, _vp, _pvp]),
    "iluamg_run_bench_trisolve": (_i, [_vp, _vp, _pvp]), "iluamg_run_schur_solve": (_i, [_vp, _vp, _pvp]),
    "iluamg_report_status": (_i, [_vp]), "iluamg_report_scalar_count": (_i, [_vp]),
    "iluamg_report_scalar_key": (_cs, [_vp, _i]), "iluamg_report_scalar_value": (_cs, [_vp, _i]),
    "iluamg_report_get": (_cs, [_vp, _cs]), "iluamg_report_table_count": (_i, [_vp]),
    "iluamg_report_table_name": (_cs, [_vp, _i]), "iluamg_report_table_csv": (_cs, [_vp, _cs]),
    "iluamg_report_json": (_cs, [_vp]), "iluamg_report_text": (_cs, [_vp]),
    "iluamg_report_free": (None, [_vp]),
    # ilug_* device handles
    "ilug_last_error": (_cs, []), "ilug_device_count": (_i, [_pi]), "ilug_set_device": (_i, [_i]),
    "ilug_synchronize": (_i, [_vp]),
    "ilug_matrix_from_csr": (_i, [_ll, _ll, _pll, _pll, _pd, _pvp]),
    "ilug_matrix_copy_csr": (_i, [_vp, _pll, _pll, _pd]),
    "ilug_ilu_factorize": (_i, [_vp, _vp, _pvp, _pvp]),
    "ilug_ilu_factorize_device": (_i, [_vp, _vp, _pvp, _pvp]),
    "ilug_matmul_device": (_i, [_vp, _vp, _pvp]), "ilug_galerkin_device": (_i, [_vp, _vp, _vp, _pvp]),
    "ilug_factors_create": (_i, [_vp, _vp, _i, _i, _i, _pvp]),
    "ilug_factors_from_csr": (_i, [_ll, _pll, _pll, _pd, _pll, _pll, _pd, _i, _i, _i, _pvp]),
    "ilug_factors_rows": (_ll, [_vp]), "ilug_factors_refactor": (_i, [_vp, _vp]), "ilug_factors_nnz": (_i, [_vp, _pll, _pll]),
    "ilug_factors_download_upper": (_i, [_vp, _pll, _pll, _pd, _pd, _pd, _pi]),
    "ilug_sweep_lower": (_i, [_vp, _vp, _vp, _ll, _vp]), "ilug_sweep_upper": (_i, [_vp, _vp, _vp, _ll, _vp]),
    "ilug_sweep_upper_host": (_i, [_vp, _pd, _pd, _ll]),
    "ilug_solve_lower": (_i, [_vp, _vp, _vp, _vp]), "ilug_solve_upper": (_i, [_vp, _vp, _vp, _vp]),
    "ilug_factors_stats": (_i, [_vp, _pll, _pll, _pll, _pll, _pi, _pi]),
    "ilug_factors_wave": (_i, [_vp, _pll, _pll, _pi, _pll]),
    "ilug_factors_free": (None, [_vp]),
    "ilug_dmatrix_create": (_i, [_vp, _pvp]), "ilug_spmv": (_i, [_vp, _vp, _vp, _vp]),
    "ilug_residual": (_i, [_vp, _vp, _vp, _vp, _vp]), "ilug_dmatrix_free": (None, [_vp]),
    "ilug_smoother_create": (_i, [_vp, _vp, _i, _pvp]), "ilug_smooth": (_i, [_vp, _vp, _vp, _pd, _vp]),
    "ilug_ilu_smooth_sweep": (_i, [_vp, _vp, _vp, _vp]), "ilug_smoother_free": (None, [_vp]),
    "ilug_smooth_host": (_i, [_vp, _pd, _pd]),
    "ilug_smooth_host_many": (_i, [_vp, _ll, _pvp, _pvp]),
    "ilug_smoother_stats": (_i, [_vp, _pll, _pll, _pll, _pll, _pll]),
    "ilug_smoother_wave": (_i, [_vp, _pll, _pll, _pi, _pll]),
    "ilug_smoother_sweeps_fused": (_i, [_vp, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp]),
    "ilug_smoother_sweep_once": (_i, [_vp, _i, _vp, _vp, _vp, _vp]),
    "ilug_hierarchy_create": (_i, [_vp, _vp, _pvp]), "ilug_hierarchy_create_host": (_i, [_vp, _vp, _pvp]),
    "ilug_hierarchy_levels": (_i, [_vp]), "ilug_hierarchy_level_matrix": (_i, [_vp, _i, _i, _pvp]),
    "ilug_hierarchy_operator_complexity": (_d, [_vp]), "ilug_vcycle": (_i, [_vp, _vp, _vp, _vp]),
    "ilug_vcycle_graph_nodes": (_ll, [_vp]), "ilug_hierarchy_free": (None, [_vp]),
    "ilug_gmres": (_i, [_vp, _vp, _vp, _vp, _pll, _pd, _vp]),
    # multi-GPU (see paper_2111_09512_b200/dist.py)
    "ilug_dist_partition": (_i, [_ll, _i, _pll]),
    "ilug_dist_generate_rows": (_i, [_cs, _ll, _ll, _pvp]),
    "ilug_dist_plan_create": (_i, [_vp, _ll, _i, _i, _pvp]),
    "ilug_dist_plan_info": (_i, [_vp, _pll, _pll, _pll]),
    "ilug_dist_plan_requests": (_ll, [_vp, _i, _pll]),
    "ilug_dist_plan_set_sends": (_i, [_vp, _i, _pll, _ll]),
    "ilug_dist_plan_sends": (_ll, [_vp, _i, _pll]),
    "ilug_dist_plan_matrix": (_i, [_vp, _i, _pvp]),
    "ilug_dist_plan_free": (None, [_vp]),
    "ilug_dist_unique_id": (_i, [_vp]),
    "ilug_dist_comm_create": (_i, [_i, _i, _vp, _pvp]),
    "ilug_dist_group_create": (_i, [_i, _pvp]), "ilug_dist_group_free": (None, [_vp]),
    "ilug_dist_group_abort": (None, [_vp]),
    "ilug_dist_comm_create_local": (_i, [_vp, _i, _pvp]),
    "ilug_dist_plan_exchange": (_i, [_vp, _vp]),
    "ilug_dist_allreduce_sum": (_i, [_vp, _vp, _ll, _vp]),
    "ilug_dist_comm_free": (None, [_vp]),
    "ilug_dist_smoother_create": (_i, [_vp, _vp, _vp, _pvp]),
    "ilug_dist_smooth": (_i, [_vp, _vp, _vp, _vp]),
    "ilug_dist_residual": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "ilug_dist_smoother_stats": (_i, [_vp, _pll, _pll, _pll, _pll]),
    "ilug_dist_smoother_free": (None, [_vp]),
    "ilug_dist_smooth_host": (_i, [_vp, _pd, _pd]),
    "ilug_dist_smooth_host_many": (_i, [_vp, _ll, _pvp, _pvp]),
    "ilug_dist_smoother_sweep_once": (_i, [_vp, _i, _vp, _vp, _vp, _vp]),
    "ilug_dist_solver_create": (_i, [_vp, _vp, _pvp]),
    "ilug_dist_gmres": (_i, [_vp, _vp, _vp, _vp, _pll, _pd, _vp]),
    "ilug_dist_vcycle": (_i, [_vp, _vp, _vp, _vp]),
    "ilug_dist_solver_info": (_i, [_vp, _pll, _pll, _pi]),
    "ilug_dist_solver_levels": (_i, [_vp]),
    "ilug_dist_solver_free": (None, [_vp]),
    "ilug_dist_level_plans": (_i, [_vp, _i, _i, _pvp]),
    "ilug_dist_levels_count": (_i, [_vp]),
    "ilug_dist_levels_plan": (_i, [_vp, _i, _i, _pvp]),
    "ilug_dist_levels_last": (_i, [_vp, _i, _pvp]),
    "ilug_dist_levels_free": (None, [_vp]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args
EXPORTED_SYMBOLS = tuple(_SIGS)


class IlugError(RuntimeError):
    """A non-zero status from the C ABI (2 invalid, 3 numeric)."""

    def __init__(self, status: int, message: str):
        super().__init__(f"[status {status}] {message}")
        self.status = status
        self.message = message


def _check(status: int, allow_not_converged: bool = False) -> int:
    if status == OK or (allow_not_converged and status == NOT_CONVERGED):
        return status
    raise IlugError(status, lib.iluamg_last_error().decode())


def _ptr(a, n: Optional[int] = None) -> Optional[int]:
    """Device address of a CUDA float64 tensor / raw int / None.

    Tensors are checked before their address crosses the C ABI: they must be
    CUDA, float64, contiguous and hold at least ``n`` elements (a CPU or short
    tensor would otherwise turn into out-of-bounds device accesses that poison
    the CUDA context). Raw integers are trusted as-is.
    """
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if hasattr(a, "data_ptr"):
        if not getattr(a, "is_cuda", False):
            raise TypeError(f"expected a CUDA tensor, got a tensor on {getattr(a, 'device', '?')}")
        if str(a.dtype) != "torch.float64":
            raise TypeError(f"expected a float64 tensor, got {a.dtype}")
        if not a.is_contiguous():
            raise ValueError("expected a contiguous tensor")
        if n is not None and a.numel() < n:
            raise ValueError(f"tensor has {a.numel()} elements, the operator needs {n}")
        return a.data_ptr()
    raise TypeError(f"cannot take a device pointer of {type(a)!r}")


def _host_ptrs(arrs, n: Optional[int] = None):
    """void*[] of host float64 arrays (numpy arrays or CPU torch tensors) of >= n elements."""
    ptrs = (C.c_void_p * max(len(arrs), 1))()
    for i, a in enumerate(arrs):
        if hasattr(a, "data_ptr"):
            if getattr(a, "is_cuda", False) or str(a.dtype) != "torch.float64" or not a.is_contiguous():
                raise TypeError("host tensors must be contiguous float64 CPU tensors")
            size = a.numel()
            ptrs[i] = a.data_ptr()
        else:
            if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
                raise TypeError("host arrays must be contiguous float64")
            size = a.size
            ptrs[i] = a.ctypes.data
        if n is not None and size < n:
            raise ValueError(f"host array has {size} elements, the operator needs {n}")
    return ptrs


def _stream(s) -> Optional[int]:
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream  # torch.cuda.Stream


def _np(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _as(arr, ctype):
    return arr.ctypes.data_as(C.POINTER(ctype))


def device_count() -> int:
    n = C.c_int(0)
    _check(lib.ilug_device_count(C.byref(n)))
    return n.value


def config_reference() -> str:
    return lib.iluamg_config_reference().decode()


class Matrix:
    """Host CSR matrix handle (iluamg_matrix)."""

    def __init__(self, handle: int):
        self.h = C.c_void_p(handle)

    @classmethod
    def generate(cls, spec: str) -> "Matrix":
        out = C.c_void_p()
        _check(lib.iluamg_matrix_generate(spec.encode(), C.byref(out)))
        return cls(out.value)

    @classmethod
    def read(cls, path: str) -> "Matrix":
        out = C.c_void_p()
        _check(lib.iluamg_matrix_read(path.encode(), C.byref(out)))
        return cls(out.value)

    @classmethod
    def from_csr(cls, nrows, ncols, row_starts, col_indices, values) -> "Matrix":
        rp, ci, v = _np(row_starts, np.int64), _np(col_indices, np.int64), _np(values, np.float64)
        out = C.c_void_p()
        _check(lib.ilug_matrix_from_csr(nrows, ncols, _as(rp, C.c_longlong), _as(ci, C.c_longlong),
                                        _as(v, C.c_double), C.byref(out)))
        return cls(out.value)

    def write(self, path: str) -> None:
        _check(lib.iluamg_matrix_write(self.h, path.encode()))

    @property
    def rows(self) -> int:
        return lib.iluamg_matrix_rows(self.h)

    @property
    def cols(self) -> int:
        return lib.iluamg_matrix_cols(self.h)

    @property
    def nnz(self) -> int:
        return lib.iluamg_matrix_nnz(self.h)

    def csr(self):
        rp = np.empty(self.rows + 1, np.int64)
        ci = np.empty(self.nnz, np.int64)
        v = np.empty(self.nnz, np.float64)
        _check(lib.ilug_matrix_copy_csr(self.h, _as(rp, C.c_longlong), _as(ci, C.c_longlong), _as(v, C.c_double)))
        return rp, ci, v

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and lib is not None:  # not at interpreter exit
            lib.iluamg_matrix_free(self.h)
            self.h = C.c_void_p()


class Config:
    """Flat dotted-key config (iluamg_config); unknown keys fail."""

    def __init__(self, **kv):
        out = C.c_void_p()
        _check(lib.iluamg_config_create(C.byref(out)))
        self.h = out
        for k, v in kv.items():
            self.set(k.replace("__", "."), v)

    def set(self, key: str, value) -> "Config":
        if isinstance(value, bool):
            value = "true" if value else "false"
        _check(lib.iluamg_config_set(self.h, key.encode(), str(value).encode()))
        return self

    def update(self, d: Dict[str, object]) -> "Config":
        for k, v in d.items():
            self.set(k, v)
        return self

    def get(self, key: str) -> Optional[str]:
        r = lib.iluamg_config_get(self.h, key.encode())
        return None if r is None else r.decode()

    def load(self, path: str) -> "Config":
        _check(lib.iluamg_config_load(self.h, path.encode()))
        return self

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and lib is not None:  # not at interpreter exit
            lib.iluamg_config_free(self.h)
            self.h = C.c_void_p()


@dataclass
class Report:
    status: int
    scalars: Dict[str, str] = field(default_factory=dict)
    order: List[str] = field(default_factory=list)
    tables: Dict[str, str] = field(default_factory=dict)
    json: str = ""
    text: str = ""

    def __getitem__(self, k: str) -> str:
        return self.scalars[k]

    def table_rows(self, name: str) -> List[Dict[str, str]]:
        lines = [l for l in self.tables[name].splitlines() if l]
        head = lines[0].split(",")
        return [dict(zip(head, l.split(","))) for l in lines[1:]]


def _report(handle: C.c_void_p, status: int) -> Report:
    r = Report(status=status)
    for i in range(lib.iluamg_report_scalar_count(handle)):
        k = lib.iluamg_report_scalar_key(handle, i).decode()
        r.scalars[k] = lib.iluamg_report_scalar_value(handle, i).decode()
        r.order.append(k)
    for i in range(lib.iluamg_report_table_count(handle)):
        name = lib.iluamg_report_table_name(handle, i).decode()
        r.tables[name] = lib.iluamg_report_table_csv(handle, name.encode()).decode()
    r.json = lib.iluamg_report_json(handle).decode()
    r.text = lib.iluamg_report_text(handle).decode()
    lib.iluamg_report_free(handle)
    return r


def _run(fn, A: Optional[Matrix], cfg: Config) -> Report:
    out = C.c_void_p()
    st = fn(A.h if A is not None else None, cfg.h, C.byref(out))
    _check(st, allow_not_converged=True)
    return _report(out, st)


def run_solve(A, cfg):
    return _run(lib.iluamg_run_solve, A, cfg)


def run_bench_trisolve(A, cfg):
    return _run(lib.iluamg_run_bench_trisolve, A, cfg)


def run_schur_solve(A, cfg):
    return _run(lib.iluamg_run_schur_solve, A, cfg)


def run_analyze(A, cfg):
    return _run(lib.iluamg_run_analyze, A, cfg)


def ilu_factorize(A: Matrix, cfg: Config):
    """Host ILU(0)/ILUT -> (L strict, U with diagonal) as Matrix handles."""
    L, U = C.c_void_p(), C.c_void_p()
    _check(lib.ilug_ilu_factorize(A.h, cfg.h, C.byref(L), C.byref(U)))
    return Matrix(L.value), Matrix(U.value)


def matmul_device(A: Matrix, B: Matrix) -> Matrix:
    """C = A B on the device (bitwise the host/reference SpGEMM)."""
    out = C.c_void_p()
    _check(lib.ilug_matmul_device(A.h, B.h, C.byref(out)))
    return Matrix(out.value)


def galerkin_device(A: Matrix, P: Matrix, R: Matrix) -> Matrix:
    """R (A P) on the device (the AMG coarse operator)."""
    out = C.c_void_p()
    _check(lib.ilug_galerkin_device(A.h, P.h, R.h, C.byref(out)))
    return Matrix(out.value)


def ilu_factorize_device(A: Matrix, cfg: Config):
    """The device objects' factorisation: ILU(0) and ILUT on the GPU."""
    L, U = C.c_void_p(), C.c_void_p()
    _check(lib.ilug_ilu_factorize_device(A.h, cfg.h, C.byref(L), C.byref(U)))
    return Matrix(L.value), Matrix(U.value)


SCALING = {"none": 0, "row": 1, "row_col": 2}
UPPER = {"scaled": 0, "jacobi": 1}


class Factors:
    """Device ILU factors (K1 scaling applied on the device)."""

    def __init__(self, handle):
        self.h = handle

    @classmethod
    def create(cls, A: Matrix, cfg: Config, scaling="row", upper="scaled", direct=False):
        out = C.c_void_p()
        _check(lib.ilug_factors_create(A.h, cfg.h, SCALING[scaling], UPPER[upper], int(direct), C.byref(out)))
        return cls(out)

    @classmethod
    def from_csr(cls, n, L, U, scaling="row", upper="scaled", direct=False):
        """L, U: (row_starts, col_indices, values) tuples."""
        Lr, Lc, Lv = (_np(L[0], np.int64), _np(L[1], np.int64), _np(L[2], np.float64))
        Ur, Uc, Uv = (_np(U[0], np.int64), _np(U[1], np.int64), _np(U[2], np.float64))
        out = C.c_void_p()
        _check(lib.ilug_factors_from_csr(n, _as(Lr, C.c_longlong), _as(Lc, C.c_longlong), _as(Lv, C.c_double),
                                         _as(Ur, C.c_longlong), _as(Uc, C.c_longlong), _as(Uv, C.c_double),
                                         SCALING[scaling], UPPER[upper], int(direct), C.byref(out)))
        return cls(out)

    @property
    def rows(self) -> int:
        return lib.ilug_factors_rows(self.h)

    def refactor(self, A: Matrix):
        """New values, same pattern (ILU(0) factors): ilug_factors_refactor."""
        _check(lib.ilug_factors_refactor(self.h, A.h))

    def stats(self):
        n, nl, nu, pad = C.c_longlong(), C.c_longlong(), C.c_longlong(), C.c_longlong()
        ll, lu = C.c_int(), C.c_int()
        _check(lib.ilug_factors_stats(self.h, C.byref(n), C.byref(nl), C.byref(nu), C.byref(pad),
                                      C.byref(ll), C.byref(lu)))
        return dict(n=n.value, nnz_Ls=nl.value, nnz_Us=nu.value, padded_Us=pad.value,
                    levels_L=ll.value, levels_U=lu.value)

    def wave(self):
        """Wavefront plan tile counts and the stalled flag (see ilug_factors_wave)."""
        tl, tu, st, wt = C.c_longlong(), C.c_longlong(), C.c_int(), C.c_longlong()
        _check(lib.ilug_factors_wave(self.h, C.byref(tl), C.byref(tu), C.byref(st), C.byref(wt)))
        return dict(tiles_L=tl.value, tiles_U=tu.value, stalled=bool(st.value), waits=wt.value)

    def download_upper(self):
        nl, nu = C.c_longlong(), C.c_longlong()
        _check(lib.ilug_factors_nnz(self.h, C.byref(nl), C.byref(nu)))
        n = self.rows
        rp = np.empty(n + 1, np.int64)
        ci = np.empty(nu.value, np.int64)
        v = np.empty(nu.value, np.float64)
        rs = np.empty(n, np.float64)
        cs = np.empty(n, np.float64)
        fl = C.c_int()
        _check(lib.ilug_factors_download_upper(self.h, _as(rp, C.c_longlong), _as(ci, C.c_longlong),
                                               _as(v, C.c_double), _as(rs, C.c_double), _as(cs, C.c_double),
                                               C.byref(fl)))
        return (rp, ci, v), (rs if fl.value & 1 else None), (cs if fl.value & 2 else None)

    def sweep_lower(self, b, y, m, stream=None):
        n = self.rows
        _check(lib.ilug_sweep_lower(self.h, _ptr(b, n), _ptr(y, n), m, _stream(stream)))

    def sweep_upper(self, b, x, m, stream=None):
        n = self.rows
        _check(lib.ilug_sweep_upper(self.h, _ptr(b, n), _ptr(x, n), m, _stream(stream)))

    def sweep_upper_host(self, b: np.ndarray, m: int) -> np.ndarray:
        b = _np(b, np.float64)
        x = np.empty_like(b)
        _check(lib.ilug_sweep_upper_host(self.h, _as(b, C.c_double), _as(x, C.c_double), m))
        return x

    def solve_lower(self, b, y, stream=None):
        n = self.rows
        _check(lib.ilug_solve_lower(self.h, _ptr(b, n), _ptr(y, n), _stream(stream)))

    def solve_upper(self, b, x, stream=None):
        n = self.rows
        _check(lib.ilug_solve_upper(self.h, _ptr(b, n), _ptr(x, n), _stream(stream)))

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and lib is not None:  # not at interpreter exit
            lib.ilug_factors_free(self.h)
            self.h = C.c_void_p()


class DeviceMatrix:
    def __init__(self, A: Matrix):
        out = C.c_void_p()
        _check(lib.ilug_dmatrix_create(A.h, C.byref(out)))
        self.h = out
        self.n, self.ncols = A.rows, A.cols

    def spmv(self, x, y, stream=None):
        _check(lib.ilug_spmv(self.h, _ptr(x, self.ncols), _ptr(y, self.n), _stream(stream)))

    def residual(self, x, b, r, stream=None):
        _check(lib.ilug_residual(self.h, _ptr(x, self.ncols), _ptr(b, self.n), _ptr(r, self.n), _stream(stream)))

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and lib is not None:  # not at interpreter exit
            lib.ilug_dmatrix_free(self.h)
            self.h = C.c_void_p()


class Smoother:
    def __init__(self, A: Matrix, cfg: Config, which: int = 0):
        out = C.c_void_p()
        _check(lib.ilug_smoother_create(A.h, cfg.h, which, C.byref(out)))
        self.h = out
        self.n = A.rows

    def smooth(self, b, x, stream=None, want_norm=False):
        nrm = C.c_double()
        _check(lib.ilug_smooth(self.h, _ptr(b, self.n), _ptr(x, self.n), C.byref(nrm) if want_norm else None,
                               _stream(stream)))
        return nrm.value if want_norm else None

    def ilu_sweep(self, b, x, stream=None):
        _check(lib.ilug_ilu_smooth_sweep(self.h, _ptr(b, self.n), _ptr(x, self.n), _stream(stream)))

    def smooth_host_many(self, bs, xs):
        """Pipelined x_i <- smooth(A, b_i, x_i) over host arrays (numpy or CPU
        tensors; pinned memory overlaps the copies), ilug_smooth_host_many."""
        if len(bs) != len(xs):
            raise ValueError("bs and xs must have the same length")
        _check(lib.ilug_smooth_host_many(self.h, len(bs), _host_ptrs(bs, self.n), _host_ptrs(xs, self.n)))

    def wave(self):
        """Wavefront plan tile counts and the stalled flag (see ilug_smoother_wave)."""
        tl, tu, st, wt = C.c_longlong(), C.c_longlong(), C.c_int(), C.c_longlong()
        _check(lib.ilug_smoother_wave(self.h, C.byref(tl), C.byref(tu), C.byref(st), C.byref(wt)))
        return dict(tiles_L=tl.value, tiles_U=tu.value, stalled=bool(st.value), waits=wt.value)

    def sweeps_fused(self, which: int, nsweeps: int, x_in, rhs, tmp, out, stream=None):
        _check(lib.ilug_smoother_sweeps_fused(self.h, which, nsweeps, _ptr(x_in, self.n), _ptr(rhs, self.n),
                                              _ptr(tmp, self.n) if tmp is not None else None, _ptr(out, self.n),
                                              _stream(stream)))

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and lib is not None:  # not at interpreter exit
            lib.ilug_smoother_free(self.h)
            self.h = C.c_void_p()


class Hierarchy:
    def __init__(self, A: Matrix, cfg: Config, host_only: bool = False):
        out = C.c_void_p()
        fn = lib.ilug_hierarchy_create_host if host_only else lib.ilug_hierarchy_create
        _check(fn(A.h, cfg.h, C.byref(out)))
        self.h = out
        self.n = A.rows

    @property
    def levels(self) -> int:
        return lib.ilug_hierarchy_levels(self.h)

    def level_matrix(self, level: int, which: str = "A") -> Matrix:
        out = C.c_void_p()
        _check(lib.ilug_hierarchy_level_matrix(self.h, level, {"A": 0, "P": 1, "R": 2}[which], C.byref(out)))
        return Matrix(out.value)

    @property
    def operator_complexity(self) -> float:
        return lib.ilug_hierarchy_operator_complexity(self.h)

    def vcycle(self, r, z, stream=None):
        _check(lib.ilug_vcycle(self.h, _ptr(r, self.n), _ptr(z, self.n), _stream(stream)))

    @property
    def graph_nodes(self) -> int:
        return lib.ilug_vcycle_graph_nodes(self.h)

    def gmres(self, cfg: Config, b, x, stream=None):
        it, rr = C.c_longlong(), C.c_double()
        st = lib.ilug_gmres(self.h, cfg.h, _ptr(b, self.n), _ptr(x, self.n), C.byref(it), C.byref(rr),
                            _stream(stream))
        _check(st, allow_not_converged=True)
        return dict(status=st, iterations=it.value, final_relres=rr.value)

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and lib is not None:  # not at interpreter exit
            lib.ilug_hierarchy_free(self.h)
            self.h = C.c_void_p()
