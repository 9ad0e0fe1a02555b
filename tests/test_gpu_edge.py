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
