"""CPU: pin the oracle before trusting it.

(a) The plain-C restatement (oracle/iluamg_oracle.c) is bitwise the reference
    library (oracle/_ref) on every hot-path kernel.
(b) Both reproduce the reference's own known-answer tests (restated from
    tests/test_trisolve.cpp, tests/acceptance.cpp) and the committed golden
    fixtures in tests/golden/ (made by tests/golden/make_golden.py from the
    reference itself).
"""
import os

import numpy as np
import pytest

from conftest import bitwise, rel_err

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def csr_of(M):
    M = np.asarray(M, dtype=np.float64)
    rp, ci, v = [0], [], []
    for row in M:
        nz = np.nonzero(row)[0]
        ci += list(nz)
        v += list(row[nz])
        rp.append(len(ci))
    return np.array(rp), np.array(ci, dtype=np.int64), np.array(v)


def random_strict(n, upper, per_row, scale, rng):
    M = np.zeros((n, n))
    for i in range(n):
        lo, hi = (i + 1, n) if upper else (0, i)
        if hi <= lo:
            continue
        p = min(1.0, per_row / (hi - lo))
        for j in range(lo, hi):
            if rng.random() < p:
                M[i, j] = scale * rng.uniform(-1, 1)
    return M


def neumann_partial_sum(T, b, m):
    acc, term = b.copy(), b.copy()
    for _ in range(1, m):
        term = -(T @ term)
        acc += term
    return acc


def nilpotency_index(T, upper):
    n = len(T)
    depth = np.ones(n, dtype=int)
    order = range(n - 1, -1, -1) if upper else range(n)
    for i in order:
        nz = np.nonzero(T[i])[0]
        if len(nz):
            depth[i] = max(depth[i], depth[nz].max() + 1)
    return int(depth.max())


# ---- (b) known answers from the reference's tests --------------------------------

def test_golden_upper_3x3(port, ref):
    """tests/test_trisolve.cpp:56-69: x = (0.375, 0.25, 0.5)."""
    U = csr_of([[2, 1, 0], [0, 2, 1], [0, 0, 2]])
    for x in (port.solve_upper_direct(U, np.ones(3)), ref.solve_upper_direct(ref.mat(*U), np.ones(3))):
        assert np.array_equal(x, [0.375, 0.25, 0.5])


def test_golden_identity_factors(port):
    """tests/test_trisolve.cpp:102-106, 127-132: L_s = 0 / U = I give b exactly."""
    b = np.array([2.0, -1.0, 7.0])
    Z = csr_of(np.zeros((3, 3)))
    assert np.array_equal(port.richardson_lower(Z, b, 1), b)
    I = csr_of(np.eye(3))
    assert np.array_equal(port.richardson_upper_scaled(I, np.ones(3), None, b, 1), b)


def test_golden_two_lower_steps_bitwise(port, ref):
    """tests/test_trisolve.cpp:116-125: two steps equal (I - L_s) b bitwise."""
    Ls = np.zeros((5, 5))
    Ls[1, 0], Ls[2, 1], Ls[3, 2], Ls[4, 3] = 0.5, -0.25, 2.0, 1.5
    b = np.arange(1.0, 6.0)
    want = b - port.spmv(csr_of(Ls), b)
    assert bitwise(port.richardson_lower(csr_of(Ls), b, 2), want)
    assert bitwise(ref.richardson_lower(ref.mat(*csr_of(Ls)), b, 2), want)


@pytest.mark.parametrize("seed", range(1, 7))
def test_richardson_is_neumann_partial_sum(port, seed):
    """tests/test_trisolve.cpp:151-165: 1e-13 for k = 1..8, n = 30*seed."""
    rng = np.random.default_rng(seed * 7)
    n = 30 * seed
    T = random_strict(n, True, 2.5, 0.3 if seed % 2 == 0 else 1.0, rng)
    U = csr_of(T + np.eye(n))
    b = rng.uniform(-1, 1, n)
    for k in range(1, 9):
        assert rel_err(port.richardson_upper_scaled(U, np.ones(n), None, b, k), neumann_partial_sum(T, b, k)) < 1e-13


def test_acceptance_c3_instances(port):
    """tests/acceptance.cpp:244-289: 100 seeded instances, Neumann at 1e-13 and the
    direct solve at the nilpotency index at 1e-10 (numpy-seeded instances)."""
    for seed in range(1, 101):
        rng = np.random.default_rng(seed)
        n = 20 + (seed * 37) % 181
        upper = seed % 2 == 0
        T = random_strict(n, upper, 2.5, 1.0 if seed % 3 == 0 else 0.35, rng)
        b = rng.uniform(-1, 1, n)
        idx = nilpotency_index(T, upper)
        if upper:
            U = csr_of(T + np.eye(n))
            it = lambda m: port.richardson_upper_scaled(U, np.ones(n), None, b, m)
            direct = port.solve_upper_direct(U, b)
        else:
            Ls = csr_of(T)
            it = lambda m: port.richardson_lower(Ls, b, m)
            direct = port.solve_lower_direct(Ls, b)
        for k in {1, 2, min(idx, 6), idx}:
            assert rel_err(it(k), neumann_partial_sum(T, b, k)) < 1e-13
        assert rel_err(it(idx), direct) < 1e-10


def test_row_scale_exactness(port):
    """tests/test_ilu.cpp:148-174: unit diagonal exactly, row_scale == diag(U)."""
    rng = np.random.default_rng(3)
    n = 40
    M = np.triu(random_strict(n, True, 3, 1.0, rng)) + np.diag(rng.uniform(0.5, 3, n) * rng.choice([-1, 1], n))
    U = csr_of(M)
    v, d = port.row_scale(U)
    rp, ci, _ = U
    for i in range(n):
        k = rp[i]
        assert ci[k] == i and v[k] == 1.0 and d[i] == M[i, i]
    vc, rs, cs = port.row_col_scale(U)
    assert np.allclose(rs * cs, np.diag(M), rtol=1e-15)


# ---- (a) port == reference, bitwise ------------------------------------------------

@pytest.mark.parametrize("spec", ["poisson3d(10,11,12)", "pressure27(8,8,8)", "cutcell(12,12,12)"])
def test_port_matches_reference(ilug, ref, port, spec):
    A = ilug.Matrix.generate(spec)
    Acsr = A.csr()
    Ar = ref.mat(*Acsr)
    fr = ref.ilu(Ar, ref.cfg())
    (Lr, Ur, _, _) = ref.factors_arrays(fr)
    rng = np.random.default_rng(9)
    n = A.rows
    b, x = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    assert bitwise(port.spmv(Acsr, x), ref.spmv(Ar, x, n))
    assert bitwise(port.residual(Acsr, x, b), ref.residual(Ar, x, b))
    assert bitwise(port.richardson_lower(Lr, b, 5), ref.richardson_lower(ref.mat(*Lr), b, 5))
    assert bitwise(port.solve_lower_direct(Lr, b), ref.solve_lower_direct(ref.mat(*Lr), b))
    assert bitwise(port.solve_upper_direct(Ur, b), ref.solve_upper_direct(ref.mat(*Ur), b))
    assert bitwise(port.gauss_seidel_sweep(Acsr, b, x), ref.gauss_seidel_sweep(Ar, b, x))
    for kind in ("row", "row_col"):
        fs = ref.scale(fr, kind)
        _, Us, rs, cs = ref.factors_arrays(fs)
        if kind == "row":
            v, d = port.row_scale(Ur)
            assert bitwise(v, Us[2]) and bitwise(d, rs)
        else:
            v, rs2, cs2 = port.row_col_scale(Ur)
            assert bitwise(v, Us[2]) and bitwise(rs2, rs) and bitwise(cs2, cs)
        for m in (1, 4):
            assert bitwise(port.richardson_upper_scaled(Us, rs, cs, b, m), ref.richardson_upper_scaled(fs, b, m))
        st = ref.smoother(Ar, ref.cfg({"smoother.kind": "ilu", "scaling": kind, "trisolve.m_lower": 3,
                                       "trisolve.m_upper": 4, "smoother.sweeps": 1}))
        want = ref.ilu_smooth_sweep(Ar, st, b, x)
        assert bitwise(port.ilu_smooth_sweep(Acsr, Lr, Us, rs, cs, b, x, 3, 4), want)
    # departure from normality (src/ilu.cpp:351-366)
    assert port.departure(Ur) == ref.departure(ref.mat(*Ur), 2)


def test_hash_unit_matches_reference(port, ref):
    for s, i in [(1, 0), (2111, 12345), (7, 2 ** 40)]:
        assert port.hash_unit(s, i) == ref.L.ref_hash_unit(s, i)


# ---- (b') committed fixtures produced by the reference ---------------------------------

def _fixtures():
    if not os.path.isdir(GOLDEN):
        return []
    return sorted(f for f in os.listdir(GOLDEN) if f.endswith(".npz"))


@pytest.mark.parametrize("name", _fixtures())
def test_port_against_golden_fixture(ilug, port, name):
    g = np.load(os.path.join(GOLDEN, name))
    A = ilug.Matrix.generate(str(g["spec"]))
    Acsr = A.csr()
    assert g["A_sha"] == __import__("hashlib").sha256(b"".join(a.tobytes() for a in Acsr)).hexdigest()
    L, U = ilug.ilu_factorize(A, ilug.Config().update(dict(zip(g["kv_keys"], g["kv_vals"]))))
    Lc, Uc = L.csr(), U.csr()
    v, d = port.row_scale(Uc)
    Us = (Uc[0], Uc[1], v)
    b = g["b"]
    assert bitwise(port.richardson_upper_scaled(Us, d, None, b, int(g["m"])), g["x_upper"])
    assert bitwise(port.richardson_lower(Lc, b, int(g["m"])), g["y_lower"])
    assert bitwise(port.solve_upper_direct(Us, b / d), g["x_upper_direct"])


@pytest.mark.parametrize("spec", ["poisson3d(9,7,5)", "pressure27(8,9,7)", "pressure27(6,5,4,77)",
                                  "cutcell(10,10,10)", "cutcell(12,9,8,5)"])
def test_oracle_3d_generators_bitwise(spec):
    """oracle/_ref's 3D generators (ref_gen3d, restated from SURVEY.md §8d on
    the reference's hash_unit) = the device build's generators, bit for bit —
    the bench's reference arm builds its input with them and never loads libilug."""
    import paper_2111_09512_b200 as ilug
    from oracle import oracle
    if not os.path.exists(oracle.REF_SO):
        pytest.skip("oracle/_ref not built")
    ref = oracle.Ref()
    got = ref.arrays(ref.gen3d(spec))
    want = ilug.Matrix.generate(spec).csr()
    for g, w in zip(got, want):
        assert np.array_equal(np.asarray(g).view(np.int64), np.asarray(w).astype(g.dtype).view(np.int64))
