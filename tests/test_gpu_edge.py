"""GPU edge cases of the hot path against the reference: non-finite inputs,
zero pivots of the scaled factor, non-finite operators inside GMRES, tiny and
empty systems. The device must fail (or propagate) exactly where the reference
does (status codes of include/iluamg.h: 2 invalid, 3 numeric;
tests/test_krylov.cpp:177-187, src/ilu.cpp:272-295)."""
import numpy as np
import pytest

from conftest import bitwise

pytestmark = pytest.mark.gpu


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _same_nonfinite(got, want):
    """NaN payloads differ between x86 and the GPU (default NaN vs canonical),
    so non-finite entries compare by class and sign, finite ones bitwise."""
    assert np.array_equal(np.isnan(got), np.isnan(want))
    inf = np.isinf(want)
    assert np.array_equal(np.isinf(got), inf) and np.array_equal(np.sign(got[inf]), np.sign(want[inf]))
    fin = np.isfinite(want)
    assert bitwise(got[fin], want[fin])


@pytest.mark.parametrize("spec", ["poisson3d(10,10,10)", "pressure27(8,8,8)"])
def test_sweeps_propagate_nan_and_inf(ilug, ref, torch_cuda, spec):
    A = ilug.Matrix.generate(spec)
    L, U = ilug.ilu_factorize(A, ilug.Config())
    Lc, Uc = L.csr(), U.csr()
    f = ilug.Factors.from_csr(A.rows, Lc, Uc, scaling="row")
    fr = ref.scale(ref.ilu(ref.mat(*A.csr()), ref.cfg({})), "row")
    b = np.random.default_rng(1).uniform(-1, 1, A.rows)
    b[5], b[A.rows // 2], b[-3] = np.nan, np.inf, -np.inf
    bd = _dev(torch_cuda, b)
    x = torch_cuda.empty_like(bd)
    for m in (1, 3, 6):
        f.sweep_upper(bd, x, m)
        _same_nonfinite(_host(x), ref.richardson_upper_scaled(fr, b, m))
        f.sweep_lower(bd, x, m)
        _same_nonfinite(_host(x), ref.richardson_lower(ref.mat(*Lc), b, m))


@pytest.mark.parametrize("scaling", ["row", "row_col"])
def test_zero_pivot_in_u_is_numeric_error(ilug, ref, torch_cuda, scaling):
    """A zero diagonal in U: the reference's row_scale/row_col_scale throw
    ErrorKind::numeric; the device K1 reports status 3 naming the same row."""
    A = ilug.Matrix.generate("poisson2d(9,7)")
    L, U = ilug.ilu_factorize(A, ilug.Config())
    Lc, (urp, uci, uv) = L.csr(), U.csr()
    uv = uv.copy()
    row = 17
    uv[urp[row]] = 0.0  # the diagonal is the first stored entry of an upper row
    assert uci[urp[row]] == row
    with pytest.raises(ilug.IlugError) as e:
        ilug.Factors.from_csr(A.rows, Lc, (urp, uci, uv), scaling=scaling)
    assert e.value.status == 3 and f"row {row}" in e.value.message
    Lh, Uh = ref.mat(*Lc), ref.mat(urp, uci, uv)
    with pytest.raises(Exception) as er:
        ref.scale(ref.factors_make(Lh, Uh), scaling)
    assert "[status 3]" in str(er.value)


def test_nan_operator_fails_like_reference(ilug, ref, torch_cuda):
    """NaN in A (tests/test_krylov.cpp:177-187): the reference's solve fails
    with a numeric error; so does the device solve."""
    A = ilug.Matrix.generate("poisson2d(8,8)")
    rp, ci, v = A.csr()
    v = v.copy()
    v[10] = np.nan
    kv = {"krylov.tol": "1e-8", "smoother.kind": "ilu", "trisolve.m_lower": 5, "trisolve.m_upper": 5}
    with pytest.raises(Exception) as er:
        ref.run_solve((rp, ci, v), kv)
    assert "[status 3]" in str(er.value)
    with pytest.raises(ilug.IlugError) as e:
        ilug.run_solve(ilug.Matrix.from_csr(A.rows, A.rows, rp, ci, v), ilug.Config().update(kv))
    assert e.value.status == 3


@pytest.mark.parametrize("spec", ["poisson2d(1,1)", "poisson2d(2,1)", "poisson2d(3,2)", "poisson3d(2,2,2)"])
def test_tiny_systems_match_reference(ilug, ref, torch_cuda, spec):
    kv = {"krylov.tol": "1e-8", "smoother.kind": "ilu", "trisolve.m_lower": 5, "trisolve.m_upper": 5}
    A = ilug.Matrix.generate(spec)
    want = ref.run_solve(A.csr(), kv)
    got = ilug.run_solve(A, ilug.Config().update(kv))
    assert got["converged"] == want["converged"] == "true"
    assert abs(int(got["iterations"]) - int(want["iterations"])) <= 1
    assert got["levels"] == want["levels"]


def test_empty_matrix_like_reference(ilug, ref, torch_cuda):
    """A 0 x 0 system: the reference returns status 0, converged after 0
    iterations, one level; the device path does the same."""
    empty = (np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0))
    want = ref.run_solve(empty, {})
    got = ilug.run_solve(ilug.Matrix.from_csr(0, 0, *empty), ilug.Config())
    for k in ("iterations", "converged", "levels"):
        assert got[k] == want[k], k


@pytest.mark.parametrize("spec", ["poisson3d(17,13,11)", "pressure27(12,12,12)", "cutcell(14,14,14)",
                                  "poisson2d(33,31)", "anisotropic2d(20,20,0.01)", "poisson2d(1,1)"])
def test_device_ilu0_bitwise(ilug, ref, torch_cuda, spec):
    """Device ILU(0) (dependency-flag scheduled) = host ILU(0) = the reference."""
    A = ilug.Matrix.generate(spec)
    cfg = ilug.Config()
    Ld, Ud = ilug.ilu_factorize_device(A, cfg)
    Lh, Uh = ilug.ilu_factorize(A, cfg)
    for d, h in ((Ld.csr(), Lh.csr()), (Ud.csr(), Uh.csr())):
        assert np.array_equal(d[0], h[0]) and np.array_equal(d[1], h[1])
        assert bitwise(d[2], h[2])
    Lr, Ur, _, _ = ref.factors_arrays(ref.ilu(ref.mat(*A.csr()), ref.cfg({})))
    assert bitwise(Ud.csr()[2], Ur[2]) and bitwise(Ld.csr()[2], Lr[2])


@pytest.mark.parametrize("patch", ["error", "replace"])
def test_device_ilu0_zero_pivot(ilug, torch_cuda, patch):
    """A structurally present but zero pivot: the same error (first row) or the
    same substituted pivot as the host path."""
    n = 6
    rp = np.arange(0, 2 * n + 1, 2)[: n + 1].astype(np.int64)
    rows, cols, vals = [], [], []
    for i in range(n):  # lower bidiagonal with a zero diagonal at row 3
        if i > 0:
            rows.append(i), cols.append(i - 1), vals.append(-1.0)
        rows.append(i), cols.append(i), vals.append(0.0 if i == 3 else 4.0)
    rp = np.zeros(n + 1, np.int64)
    for r in rows:
        rp[r + 1] += 1
    rp = np.cumsum(rp)
    A = ilug.Matrix.from_csr(n, n, rp, np.array(cols, np.int64), np.array(vals))
    cfg = ilug.Config().set("ilu.pivot_patch", patch)
    if patch == "error":
        for fn in (ilug.ilu_factorize, ilug.ilu_factorize_device):
            with pytest.raises(ilug.IlugError) as e:
                fn(A, cfg)
            assert e.value.status == 3 and "step 3" in e.value.message
    else:
        Ld, Ud = ilug.ilu_factorize_device(A, cfg)
        Lh, Uh = ilug.ilu_factorize(A, cfg)
        assert bitwise(Ud.csr()[2], Uh.csr()[2]) and bitwise(Ld.csr()[2], Lh.csr()[2])


def test_device_ilu0_large_bitwise(ilug, torch_cuda):
    """2.1 M rows (deep DAG, many blocks waiting on earlier ones): bitwise."""
    A = ilug.Matrix.generate("pressure27(128,128,128)")
    cfg = ilug.Config()
    Ld, Ud = ilug.ilu_factorize_device(A, cfg)
    Lh, Uh = ilug.ilu_factorize(A, cfg)
    assert bitwise(Ud.csr()[2], Uh.csr()[2]) and bitwise(Ld.csr()[2], Lh.csr()[2])


@pytest.mark.parametrize("kind", ["gauss_seidel", "ilu", "poly_gs"])
def test_setup_pipeline_errors_propagate(ilug, ref, torch_cuda, kind):
    """A failure inside the overlapped setup (the device builder thread for a
    GS smoother with a zero diagonal, the early factorisation thread for an ILU
    zero pivot, the poly-GS inverted diagonal computed on the device from the
    AMG setup's copy of A) surfaces as the reference's status-3 error, and the
    next solve in the process still works."""
    A = ilug.Matrix.generate("poisson2d(16,16)")
    rp, ci, v = A.csr()
    v = v.copy()
    row = 37
    for k in range(rp[row], rp[row + 1]):
        if ci[k] == row:
            v[k] = 0.0  # structurally present, numerically zero diagonal
    kv = {"krylov.tol": "1e-8", "smoother.kind": kind, "amg.coarsening": "pmis", "amg.coarse_size": "16"}
    with pytest.raises(Exception) as er:
        ref.run_solve((rp, ci, v), kv)
    assert "[status 3]" in str(er.value)
    with pytest.raises(ilug.IlugError) as e:
        ilug.run_solve(ilug.Matrix.from_csr(A.rows, A.rows, rp, ci, v), ilug.Config().update(kv))
    assert e.value.status == 3
    ok = ilug.run_solve(A, ilug.Config().update(kv))
    assert ok["converged"] == "true"
