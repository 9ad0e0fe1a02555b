"""ORACLE / TEST INFRASTRUCTURE ONLY — the checker, never the product.

ctypes views of
  * ``oracle/_ref/libiluamg_ref.so``: the unmodified reference (iluamg) compiled
    from /root/reference/proj/src plus ``ref_shim.cpp`` (see oracle/Makefile);
  * ``oracle/_build/liboracle_port.so``: the plain-C restatement
    ``oracle/iluamg_oracle.c`` (hot-path kernels only), which works where the
    reference sources are absent.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Dict, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libiluamg_ref.so")
PORT_SO = os.path.join(HERE, "_build", "liboracle_port.so")

_vp, _i, _ll, _d, _u64 = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_uint64
_pvp, _pll, _pd, _pi = C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_int)


def build(ref: bool = True) -> None:
    """Compile the port (always) and the reference (when its sources exist)."""
    targets = ["port"] + (["ref"] if ref and os.path.isdir("/root/reference/proj/src") else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class RefError(RuntimeError):
    pass


class Ref:
    """The reference library itself (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.L = C.CDLL(path)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_mat_from_csr": (_i, [_ll, _ll, _pll, _pll, _pd, _pvp]),
            "ref_mat_generate": (_i, [C.c_char_p, _pvp]), "ref_mat_read": (_i, [C.c_char_p, _pvp]),
            "ref_mat_write": (_i, [_vp, C.c_char_p]),
            "ref_mat_info": (None, [_vp, _pll, _pll, _pll]), "ref_mat_copy": (None, [_vp, _pll, _pll, _pd]),
            "ref_mat_free": (None, [_vp]), "ref_cfg_create": (_vp, []),
            "ref_cfg_set": (_i, [_vp, C.c_char_p, C.c_char_p]), "ref_cfg_free": (None, [_vp]),
            "ref_spmv": (_i, [_vp, _pd, _pd]), "ref_residual": (_i, [_vp, _pd, _pd, _pd]),
            "ref_richardson_lower": (_i, [_vp, _pd, _ll, _pd]),
            "ref_solve_lower_direct": (_i, [_vp, _pd, _pd]), "ref_solve_upper_direct": (_i, [_vp, _pd, _pd]),
            "ref_gauss_seidel_sweep": (_i, [_vp, _pd, _pd]), "ref_departure": (_i, [_vp, _i, _pd]),
            "ref_ilu_factor": (_i, [_vp, _vp, _pvp]), "ref_factors_make": (_i, [_vp, _vp, _pd, _pd, _pvp]),
            "ref_factors_scale": (_i, [_vp, _i, _pvp]), "ref_factors_L": (_vp, [_vp]),
            "ref_factors_U": (_vp, [_vp]), "ref_factors_scales": (_i, [_vp, _pd, _pd]),
            "ref_factors_free": (None, [_vp]),
            "ref_richardson_upper_scaled": (_i, [_vp, _pd, _ll, _pd]),
            "ref_solve_upper_scaled_direct": (_i, [_vp, _pd, _pd]),
            "ref_smoother_build": (_i, [_vp, _vp, _i, _pvp]), "ref_smooth": (_i, [_vp, _vp, _pd, _pd, _pd]),
            "ref_ilu_smooth_sweep": (_i, [_vp, _vp, _pd, _pd]), "ref_smoother_factors": (_vp, [_vp]),
            "ref_smoother_schur": (_vp, [_vp]), "ref_smoother_free": (None, [_vp]),
            "ref_amg_setup": (_i, [_vp, _vp, _pvp]), "ref_amg_nlevels": (_ll, [_vp]),
            "ref_amg_level_mat": (_vp, [_vp, _ll, _i]), "ref_amg_vcycle": (_i, [_vp, _pd, _pd]),
            "ref_amg_operator_complexity": (_d, [_vp]), "ref_amg_free": (None, [_vp]),
            "ref_krylov_solve": (_i, [_vp, _vp, _vp, _pd, _pd, _pll, _pi, _pd, _pd, _ll, _pll, _pd]),
            "ref_gen3d": (_i, [_i, _ll, _ll, _ll, _u64, _pvp]),
            "ref_smoother_factor_nnz": (None, [_vp, _pll, _pll, _pll]),
            "ref_dist_setup": (_i, [_vp, _vp, _i, _pvp]), "ref_dist_free": (None, [_vp]),
            "ref_dist_nlevels": (_ll, [_vp]), "ref_dist_vcycle": (_i, [_vp, _pd, _pd]),
            "ref_dist_smooth": (_i, [_vp, _ll, _pd, _pd]),
            "ref_dist_krylov": (_i, [_vp, _vp, _vp, _pd, _pd, _pll, _pi, _pd]),
            "ref_make_rhs": (_i, [_vp, _vp, _pd]), "ref_random_uniform": (None, [_ll, _u64, _pd]),
            "ref_hash_unit": (_d, [_u64, _u64]),
            "ref_time_richardson_upper": (_i, [_vp, _pd, _ll, _ll, _pd]),
            "ref_time_smooth": (_i, [_vp, _vp, _pd, _ll, _pd]),
            "ref_run_solve": (_i, [_vp, _vp, _pvp]), "ref_report_get": (C.c_char_p, [_vp, C.c_char_p]),
            "ref_run_analyze": (_i, [_vp, _vp, _pvp]),
            "ref_report_status": (_i, [_vp]), "ref_report_table_csv": (_vp, [_vp, C.c_char_p]),
            "ref_free_str": (None, [_vp]), "ref_report_free": (None, [_vp]),
            "iluamg_matrix_generate": (_i, [C.c_char_p, _pvp]), "iluamg_config_create": (_i, [_pvp]),
            "iluamg_config_set": (_i, [_vp, C.c_char_p, C.c_char_p]),
            "iluamg_run_solve": (_i, [_vp, _vp, _pvp]), "iluamg_report_get": (C.c_char_p, [_vp, C.c_char_p]),
            "iluamg_report_table_csv": (C.c_char_p, [_vp, C.c_char_p]),
            "iluamg_report_free": (None, [_vp]), "iluamg_config_free": (None, [_vp]),
            "iluamg_matrix_free": (None, [_vp]), "iluamg_last_error": (C.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args

    # -- helpers
    def _ok(self, st):
        if st != 0:
            raise RefError(f"[status {st}] {self.L.ref_last_error().decode()}")

    def mat(self, rp, ci, v, nrows=None, ncols=None):
        rp, ci, v = _i64(rp), _i64(ci), _f64(v)
        n = len(rp) - 1 if nrows is None else nrows
        out = C.c_void_p()
        self._ok(self.L.ref_mat_from_csr(n, n if ncols is None else ncols, _p(rp, C.c_int64),
                                         _p(ci, C.c_int64), _p(v, C.c_double), C.byref(out)))
        return out

    def read(self, path):
        """The reference's own Matrix Market reader (src/matrix_market.cpp)."""
        out = C.c_void_p()
        self._ok(self.L.ref_mat_read(path.encode(), C.byref(out)))
        return out

    def write(self, h, path):
        """The reference's own Matrix Market writer."""
        self._ok(self.L.ref_mat_write(h, path.encode()))

    def gen3d(self, spec):
        """Oracle-side 3D generators (poisson3d / pressure27 / cutcell specs, the
        device build's generator grammar) -> reference SparseMatrix handle."""
        kind, args = spec.split("(", 1)
        vals = [a.strip() for a in args.rstrip(")").split(",")]
        k = {"poisson3d": 0, "pressure27": 1, "cutcell": 2}[kind.strip()]
        nx, ny, nz = (int(v) for v in vals[:3])
        seed = int(vals[3]) if len(vals) > 3 else 2111
        out = C.c_void_p()
        self._ok(self.L.ref_gen3d(k, nx, ny, nz, seed, C.byref(out)))
        return out

    def generate(self, spec):
        out = C.c_void_p()
        self._ok(self.L.ref_mat_generate(spec.encode(), C.byref(out)))
        return out

    def arrays(self, h):
        nr, nc, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        self.L.ref_mat_info(h, C.byref(nr), C.byref(nc), C.byref(nnz))
        rp, ci, v = np.empty(nr.value + 1, np.int64), np.empty(nnz.value, np.int64), np.empty(nnz.value)
        self.L.ref_mat_copy(h, _p(rp, C.c_int64), _p(ci, C.c_int64), _p(v, C.c_double))
        return rp, ci, v

    def free_mat(self, h):
        self.L.ref_mat_free(h)

    def cfg(self, kv: Optional[Dict[str, object]] = None):
        h = self.L.ref_cfg_create()
        for k, val in (kv or {}).items():
            if isinstance(val, bool):
                val = "true" if val else "false"
            self._ok(self.L.ref_cfg_set(h, k.encode(), str(val).encode()))
        return C.c_void_p(h)

    def _vec_op(self, fn, h, *vecs, n):
        out = np.empty(n)
        args = [_p(_f64(v), C.c_double) for v in vecs]
        self._ok(fn(h, *args, _p(out, C.c_double)))
        return out

    # -- kernels
    def spmv(self, A, x, n):
        return self._vec_op(self.L.ref_spmv, A, x, n=n)

    def residual(self, A, x, b):
        return self._vec_op(self.L.ref_residual, A, x, b, n=len(b))

    def richardson_lower(self, L, b, m):
        b = _f64(b)
        y = np.empty_like(b)
        self._ok(self.L.ref_richardson_lower(L, _p(b, C.c_double), m, _p(y, C.c_double)))
        return y

    def solve_lower_direct(self, L, b):
        return self._vec_op(self.L.ref_solve_lower_direct, L, b, n=len(b))

    def solve_upper_direct(self, U, b):
        return self._vec_op(self.L.ref_solve_upper_direct, U, b, n=len(b))

    def gauss_seidel_sweep(self, A, b, x):
        b, x = _f64(b), _f64(x).copy()
        self._ok(self.L.ref_gauss_seidel_sweep(A, _p(b, C.c_double), _p(x, C.c_double)))
        return x

    def departure(self, T, shape):
        d = C.c_double()
        self._ok(self.L.ref_departure(T, shape, C.byref(d)))
        return d.value

    # -- factors
    def ilu(self, A, cfg):
        out = C.c_void_p()
        self._ok(self.L.ref_ilu_factor(A, cfg, C.byref(out)))
        return out

    def factors_make(self, Lh, Uh, rs=None, cs=None):
        out = C.c_void_p()
        rsp = _p(_f64(rs), C.c_double) if rs is not None else None
        csp = _p(_f64(cs), C.c_double) if cs is not None else None
        self._ok(self.L.ref_factors_make(Lh, Uh, rsp, csp, C.byref(out)))
        return out

    def scale(self, f, kind):
        out = C.c_void_p()
        self._ok(self.L.ref_factors_scale(f, {"none": 0, "row": 1, "row_col": 2}[kind], C.byref(out)))
        return out

    def factors_arrays(self, f):
        Lh, Uh = C.c_void_p(self.L.ref_factors_L(f)), C.c_void_p(self.L.ref_factors_U(f))
        L, U = self.arrays(Lh), self.arrays(Uh)
        self.free_mat(Lh)
        self.free_mat(Uh)
        n = len(U[0]) - 1
        rs, cs = np.empty(n), np.empty(n)
        fl = self.L.ref_factors_scales(f, _p(rs, C.c_double), _p(cs, C.c_double))
        return L, U, (rs if fl & 1 else None), (cs if fl & 2 else None)

    def richardson_upper_scaled(self, f, b, m):
        b = _f64(b)
        x = np.empty_like(b)
        self._ok(self.L.ref_richardson_upper_scaled(f, _p(b, C.c_double), m, _p(x, C.c_double)))
        return x

    def solve_upper_scaled_direct(self, f, b):
        return self._vec_op(self.L.ref_solve_upper_scaled_direct, f, b, n=len(b))

    # -- smoothers / AMG / Krylov
    def smoother(self, A, cfg, which=0):
        out = C.c_void_p()
        self._ok(self.L.ref_smoother_build(A, cfg, which, C.byref(out)))
        return out

    def smooth(self, A, st, b, x):
        b, x = _f64(b), _f64(x).copy()
        r = C.c_double()
        self._ok(self.L.ref_smooth(A, st, _p(b, C.c_double), _p(x, C.c_double), C.byref(r)))
        return x, r.value

    def ilu_smooth_sweep(self, A, st, b, x):
        b, x = _f64(b), _f64(x).copy()
        self._ok(self.L.ref_ilu_smooth_sweep(A, st, _p(b, C.c_double), _p(x, C.c_double)))
        return x

    def amg(self, A, cfg):
        out = C.c_void_p()
        self._ok(self.L.ref_amg_setup(A, cfg, C.byref(out)))
        return out

    def amg_levels(self, h):
        return self.L.ref_amg_nlevels(h)

    def amg_level(self, h, k, which="A"):
        m = C.c_void_p(self.L.ref_amg_level_mat(h, k, {"A": 0, "P": 1, "R": 2}[which]))
        a = self.arrays(m)
        self.free_mat(m)
        return a

    def vcycle(self, h, b, x):
        b, x = _f64(b), _f64(x).copy()
        self._ok(self.L.ref_amg_vcycle(h, _p(b, C.c_double), _p(x, C.c_double)))
        return x

    def krylov(self, A, h, cfg, b, max_hist=512):
        b = _f64(b)
        x = np.empty_like(b)
        it, conv, rr = C.c_int64(), C.c_int(), C.c_double()
        hist = np.empty(3 * max_hist)
        nh, secs = C.c_int64(), C.c_double()
        self._ok(self.L.ref_krylov_solve(A, h, cfg, _p(b, C.c_double), _p(x, C.c_double), C.byref(it),
                                         C.byref(conv), C.byref(rr), _p(hist, C.c_double), max_hist,
                                         C.byref(nh), C.byref(secs)))
        return dict(x=x, iterations=it.value, converged=bool(conv.value), final_relres=rr.value,
                    history=hist[: 3 * nh.value].reshape(-1, 3), seconds=secs.value)

    # -- composed oracle of the p-rank row-block distributed solve (block smoothers)
    def dist_setup(self, A, cfg, p):
        out = C.c_void_p()
        self._ok(self.L.ref_dist_setup(A, cfg, p, C.byref(out)))
        return out

    def dist_vcycle(self, d, b, x):
        b, x = _f64(b), _f64(x).copy()
        self._ok(self.L.ref_dist_vcycle(d, _p(b, C.c_double), _p(x, C.c_double)))
        return x

    def dist_smooth(self, d, k, b, x):
        b, x = _f64(b), _f64(x).copy()
        self._ok(self.L.ref_dist_smooth(d, k, _p(b, C.c_double), _p(x, C.c_double)))
        return x

    def dist_krylov(self, A, d, cfg, b):
        b = _f64(b)
        x = np.empty_like(b)
        it, conv, rr = C.c_int64(), C.c_int(), C.c_double()
        self._ok(self.L.ref_dist_krylov(A, d, cfg, _p(b, C.c_double), _p(x, C.c_double), C.byref(it),
                                        C.byref(conv), C.byref(rr)))
        return dict(x=x, iterations=it.value, converged=bool(conv.value), final_relres=rr.value)

    def make_rhs(self, cfg, A, n):
        b = np.empty(n)
        self._ok(self.L.ref_make_rhs(cfg, A, _p(b, C.c_double)))
        return b

    def random_uniform(self, n, seed):
        v = np.empty(n)
        self.L.ref_random_uniform(n, seed, _p(v, C.c_double))
        return v

    def time_richardson_upper(self, f, b, m, reps):
        b = _f64(b)
        s = C.c_double()
        self._ok(self.L.ref_time_richardson_upper(f, _p(b, C.c_double), m, reps, C.byref(s)))
        return s.value

    def run_solve(self, A, kv, keys=("iterations", "converged", "final_relres", "setup_seconds",
                                      "solve_seconds", "levels", "operator_complexity")):
        """The reference's own driver, run_solve (src/driver.cpp:239-260) — the body of
        iluamg_run_solve (src/capi.cpp:166-168) — on a matrix given either as a
        reference generator spec string or as (row_starts, col_indices, values)."""
        if isinstance(A, str):
            Ah = self.generate(A)
        else:
            Ah = self.mat(*A)
        cfg = self.cfg(kv)
        rep = C.c_void_p()
        try:
            self._ok(self.L.ref_run_solve(Ah, cfg, C.byref(rep)))
        finally:
            self.free_mat(Ah)
            self.L.ref_cfg_free(cfg)
        out = {k: self.L.ref_report_get(rep, k.encode()).decode() for k in keys}
        out["status"] = self.L.ref_report_status(rep)
        p = self.L.ref_report_table_csv(rep, b"history")
        out["history"] = C.cast(p, C.c_char_p).value.decode()
        self.L.ref_free_str(p)
        self.L.ref_report_free(rep)
        return out


def _analyze(self, A, kv, keys=("dep_L", "dep_U", "dep_U_row", "dep_U_rowcol", "cond_L", "cond_U",
                                 "striping_flagged", "nnz_L", "nnz_U")):
    """The reference's run_analyze (src/driver.cpp:92-163) on (rp, ci, v)."""
    Ah = self.mat(*A)
    cfg = self.cfg(kv)
    rep = C.c_void_p()
    try:
        self._ok(self.L.ref_run_analyze(Ah, cfg, C.byref(rep)))
    finally:
        self.free_mat(Ah)
        self.L.ref_cfg_free(cfg)
    out = {k: self.L.ref_report_get(rep, k.encode()).decode() for k in keys}
    self.L.ref_report_free(rep)
    return out


Ref.run_analyze = _analyze


class Port:
    """The plain-C restatement (oracle/iluamg_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.L = C.CDLL(path)
        for name in ("orc_spmv", "orc_residual", "orc_richardson_lower", "orc_richardson_upper_scaled",
                     "orc_jacobi_upper", "orc_solve_lower_direct", "orc_ilu_smooth_sweep", "orc_dense_lu_solve"):
            getattr(self.L, name).restype = None
        for name in ("orc_row_scale", "orc_row_col_scale", "orc_solve_upper_direct", "orc_gauss_seidel_sweep",
                     "orc_dense_lu"):
            getattr(self.L, name).restype = C.c_int64
        self.L.orc_departure.restype = C.c_double
        self.L.orc_hash_unit.restype = C.c_double
        self.L.orc_hash_unit.argtypes = [C.c_uint64, C.c_uint64]

    @staticmethod
    def _csr(M):
        rp, ci, v = M
        rp, ci, v = _i64(rp), _i64(ci), _f64(v)
        return rp, ci, v, (_p(rp, C.c_int64), _p(ci, C.c_int64), _p(v, C.c_double))

    def spmv(self, M, x):
        rp, ci, v, a = self._csr(M)
        x = _f64(x)
        y = np.empty(len(rp) - 1)
        self.L.orc_spmv(C.c_int64(len(rp) - 1), *a, _p(x, C.c_double), _p(y, C.c_double))
        return y

    def residual(self, M, x, b):
        rp, ci, v, a = self._csr(M)
        x, b = _f64(x), _f64(b)
        r = np.empty(len(rp) - 1)
        self.L.orc_residual(C.c_int64(len(rp) - 1), *a, _p(x, C.c_double), _p(b, C.c_double), _p(r, C.c_double))
        return r

    def richardson_lower(self, Ls, b, m):
        rp, ci, v, a = self._csr(Ls)
        b = _f64(b)
        y = np.empty_like(b)
        self.L.orc_richardson_lower(C.c_int64(len(rp) - 1), *a, _p(b, C.c_double), C.c_int64(m), _p(y, C.c_double))
        return y

    def richardson_upper_scaled(self, U, rs, cs, b, m):
        rp, ci, v, a = self._csr(U)
        b, rs = _f64(b), _f64(rs)
        csp = _p(_f64(cs), C.c_double) if cs is not None else None
        x = np.empty_like(b)
        self.L.orc_richardson_upper_scaled(C.c_int64(len(rp) - 1), *a, _p(rs, C.c_double), csp, _p(b, C.c_double),
                                           C.c_int64(m), _p(x, C.c_double))
        return x

    def jacobi_upper(self, U, b, m):
        rp, ci, v, a = self._csr(U)
        b = _f64(b)
        x = np.empty_like(b)
        self.L.orc_jacobi_upper(C.c_int64(len(rp) - 1), *a, _p(b, C.c_double), C.c_int64(m), _p(x, C.c_double))
        return x

    def row_scale(self, U):
        rp, ci, v, a = self._csr(U)
        n = len(rp) - 1
        out, d = np.empty_like(v), np.empty(n)
        bad = self.L.orc_row_scale(C.c_int64(n), *a, _p(out, C.c_double), _p(d, C.c_double))
        if bad >= 0:
            raise RefError(f"row_scale: zero diagonal entry in U at row {bad}")
        return out, d

    def row_col_scale(self, U):
        rp, ci, v, a = self._csr(U)
        n = len(rp) - 1
        out, rs, cs = np.empty_like(v), np.empty(n), np.empty(n)
        bad = self.L.orc_row_col_scale(C.c_int64(n), *a, _p(out, C.c_double), _p(rs, C.c_double), _p(cs, C.c_double))
        if bad >= 0:
            raise RefError(f"row_col_scale: zero diagonal entry in U at row {bad}")
        return out, rs, cs

    def solve_lower_direct(self, Ls, b):
        rp, ci, v, a = self._csr(Ls)
        b = _f64(b)
        x = np.empty_like(b)
        self.L.orc_solve_lower_direct(C.c_int64(len(rp) - 1), *a, _p(b, C.c_double), _p(x, C.c_double))
        return x

    def solve_upper_direct(self, U, b):
        rp, ci, v, a = self._csr(U)
        b = _f64(b)
        x = np.empty_like(b)
        bad = self.L.orc_solve_upper_direct(C.c_int64(len(rp) - 1), *a, _p(b, C.c_double), _p(x, C.c_double))
        if bad >= 0:
            raise RefError(f"solve_upper_direct: zero diagonal at row {bad}")
        return x

    def gauss_seidel_sweep(self, A, b, x):
        rp, ci, v, a = self._csr(A)
        b, x = _f64(b), _f64(x).copy()
        bad = self.L.orc_gauss_seidel_sweep(C.c_int64(len(rp) - 1), *a, _p(b, C.c_double), _p(x, C.c_double))
        if bad >= 0:
            raise RefError(f"gauss_seidel_sweep: zero diagonal at row {bad}")
        return x

    def ilu_smooth_sweep(self, A, Ls, U, rs, cs, b, x, mL, mU, direct=False):
        _, _, _, aa = self._csr(A)
        _, _, _, la = self._csr(Ls)
        _, _, _, ua = self._csr(U)
        n = len(b)
        b, x, rs = _f64(b), _f64(x).copy(), _f64(rs)
        csp = _p(_f64(cs), C.c_double) if cs is not None else None
        self.L.orc_ilu_smooth_sweep(C.c_int64(n), *aa, *la, *ua, _p(rs, C.c_double), csp, C.c_int(int(direct)),
                                    C.c_int64(mL), C.c_int64(mU), _p(b, C.c_double), _p(x, C.c_double))
        return x

    def departure(self, T):
        rp, ci, v, a = self._csr(T)
        return self.L.orc_departure(C.c_int64(len(rp) - 1), *a)

    def hash_unit(self, seed, i):
        return self.L.orc_hash_unit(seed, i)
