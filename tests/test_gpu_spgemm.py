"""Device SpGEMM and Galerkin product (kernels/spgemm.cu) against the host
SpGEMM and the reference's AMG hierarchy: bitwise equal coarse operators on
every level, exact-zero drops, NaN propagation, rows that overflow the first
hash-table size, empty rows and rectangular operands."""
import numpy as np
import pytest

from conftest import bitwise

pytestmark = pytest.mark.gpu


def _same(M, N):
    a, b = M.csr(), N.csr()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert bitwise(a[2], b[2])


@pytest.mark.parametrize("spec,kv", [
    ("pressure27(24,22,20)", {"amg.coarsening": "pmis"}),
    ("poisson3d(30,28,26)", {"amg.coarsening": "pmis"}),
    ("cutcell(24,24,24)", {"amg.coarsening": "pmis"}),
    ("anisotropic2d(60,50,0.01)", {}),
    ("stencil27(20,20,20)", {"amg.interpolation": "mm_ext", "amg.coarsening": "pmis"}),
])
def test_galerkin_every_level_bitwise(ilug, ref, torch_cuda, spec, kv):
    """R (A P) on the device reproduces every coarse operator of the host
    hierarchy (itself bitwise the reference's, tests/test_host_setup.py)."""
    A = ilug.Matrix.generate(spec)
    H = ilug.Hierarchy(A, ilug.Config().update(kv), host_only=True)
    for k in range(H.levels - 1):
        Ak, P, R = (H.level_matrix(k, w) for w in ("A", "P", "R"))
        _same(ilug.galerkin_device(Ak, P, R), H.level_matrix(k + 1, "A"))
        _same(ilug.matmul_device(Ak, P), ilug.Matrix.from_csr(*_host_matmul(Ak, P)))


def _host_matmul(A, B):
    """Dense-accumulator product in the reference's order (numpy, small sizes)."""
    arp, aci, av = A.csr()
    brp, bci, bv = B.csr()
    n = A.rows
    rows, cols, vals = [0], [], []
    acc = {}
    for i in range(n):
        acc.clear()
        for ka in range(arp[i], arp[i + 1]):
            k, a = aci[ka], av[ka]
            for kb in range(brp[k], brp[k + 1]):
                j = int(bci[kb])
                acc[j] = acc.get(j, 0.0) + a * bv[kb]
        for j in sorted(acc):
            if acc[j] != 0.0:
                cols.append(j), vals.append(acc[j])
        rows.append(len(cols))
    return n, B.cols, np.array(rows, np.int64), np.array(cols, np.int64), np.array(vals)


def _csr(n, m, dense):
    rp, ci, v = [0], [], []
    for i in range(n):
        nz = np.nonzero(dense[i])[0]
        ci.extend(nz), v.extend(dense[i, nz])
        rp.append(len(ci))
    return np.array(rp, np.int64), np.array(ci, np.int64), np.array(v, float)


def test_matmul_random_rectangular_and_cancellation(ilug, torch_cuda):
    """Random rectangular operands with exact cancellations (dropped), NaN
    (kept) and empty rows; one dense row with more distinct columns than the
    first hash table holds (overflow retry)."""
    rng = np.random.default_rng(3)
    n, k, m = 300, 700, 5000
    Ad = (rng.random((n, k)) < 0.02) * rng.integers(-3, 4, (n, k)).astype(float)
    Bd = (rng.random((k, m)) < 0.01) * rng.integers(-3, 4, (k, m)).astype(float)
    Ad[5] = 0.0                       # empty row
    Ad[7, :] = 1.0                    # a row touching ~all of B: > 512 distinct columns
    Bd[11, 13] = np.nan               # NaN propagates (kept)
    Ad[9, 11] = 1.0
    A = ilug.Matrix.from_csr(n, k, *_csr(n, k, Ad))
    B = ilug.Matrix.from_csr(k, m, *_csr(k, m, Bd))
    got = ilug.matmul_device(A, B).csr()
    want = _host_matmul(A, B)
    assert np.array_equal(got[0], want[2]) and np.array_equal(got[1], want[3])
    g, w = got[2], want[4]
    assert np.array_equal(np.isnan(g), np.isnan(w))
    fin = ~np.isnan(w)
    assert bitwise(g[fin], w[fin])


def test_run_solve_device_galerkin_matches_host(ilug, ref, torch_cuda, monkeypatch):
    """run_solve with the device Galerkin products (ILUG_GALERKIN_DEVICE=1) and
    with the host ones (default): same hierarchy, same iterations and final
    residual bits; iterations within 1 of the reference."""
    A = ilug.Matrix.generate("pressure27(32,32,32)")
    kv = {"smoother.kind": "ilu", "ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5",
          "amg.coarsening": "pmis", "krylov.tol": "1e-8"}
    monkeypatch.setenv("ILUG_GALERKIN_DEVICE", "1")
    dev = ilug.run_solve(A, ilug.Config().update(kv))
    monkeypatch.delenv("ILUG_GALERKIN_DEVICE")
    host = ilug.run_solve(A, ilug.Config().update(kv))
    for key in ("iterations", "levels", "operator_complexity", "final_relres"):
        assert dev[key] == host[key], key
    want = ref.run_solve(A.csr(), kv)
    assert abs(int(dev["iterations"]) - int(want["iterations"])) <= 1
