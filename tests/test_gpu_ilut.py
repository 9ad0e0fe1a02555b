"""Device ILUT (kernels/ilut.cu) against the host ILUT and the reference's own
ilut (src/ilu.cpp:120-265): identical patterns, bitwise identical values, same
zero-pivot errors, across drop tolerances, fill caps, matrix families and the
shared-memory capacity relaunch path."""
import numpy as np
import pytest

from conftest import bitwise

pytestmark = pytest.mark.gpu


def _same(dev, host):
    for d, h in ((dev[0].csr(), host[0].csr()), (dev[1].csr(), host[1].csr())):
        assert np.array_equal(d[0], h[0]), "row starts"
        assert np.array_equal(d[1], h[1]), "columns"
        assert bitwise(d[2], h[2]), "values"


def _ilut_cfg(ilug, droptol, lfill, patch="error"):
    return ilug.Config().update({"ilu.variant": "ilut", "ilu.droptol": repr(droptol), "ilu.lfill": str(lfill),
                                 "ilu.pivot_patch": patch})


@pytest.mark.parametrize("spec", ["poisson3d(17,13,11)", "pressure27(12,12,12)", "cutcell(14,14,14)",
                                  "poisson2d(33,31)", "anisotropic2d(20,20,0.01)", "poisson2d(1,1)",
                                  "stencil27(9,7,5)"])
@pytest.mark.parametrize("droptol,lfill", [(1e-3, 5), (0.0, 0), (1e-2, 2), (0.0, 40), (1e-1, 1)])
def test_device_ilut_bitwise(ilug, ref, torch_cuda, spec, droptol, lfill):
    A = ilug.Matrix.generate(spec)
    cfg = _ilut_cfg(ilug, droptol, lfill)
    _same(ilug.ilu_factorize_device(A, cfg), ilug.ilu_factorize(A, cfg))
    kv = {"ilu.variant": "ilut", "ilu.droptol": repr(droptol), "ilu.lfill": str(lfill)}
    Lr, Ur, _, _ = ref.factors_arrays(ref.ilu(ref.mat(*A.csr()), ref.cfg(kv)))
    Ld, Ud = ilug.ilu_factorize_device(A, cfg)
    assert np.array_equal(Ud.csr()[1], Ur[1]) and np.array_equal(Ld.csr()[1], Lr[1])
    assert bitwise(Ud.csr()[2], Ur[2]) and bitwise(Ld.csr()[2], Lr[2])


def _random_csr(rng, n, density, diag=True):
    M = (rng.random((n, n)) < density) * rng.standard_normal((n, n))
    if diag:
        M[np.arange(n), np.arange(n)] += n * 0.5 + 1.0
    rp = np.zeros(n + 1, np.int64)
    cols, vals = [], []
    for i in range(n):
        nz = np.nonzero(M[i])[0]
        cols.extend(nz), vals.extend(M[i, nz])
        rp[i + 1] = rp[i] + len(nz)
    return rp, np.array(cols, np.int64), np.array(vals)


@pytest.mark.parametrize("n,density,lfill", [(300, 0.9, 5), (700, 0.6, 30), (1300, 0.3, 3)])
def test_device_ilut_capacity_relaunch(ilug, torch_cuda, n, density, lfill):
    """Working rows longer than the first shared-memory capacity (256, then
    1024 entries): the kernel flags the overflow and the host relaunches with a
    larger capacity; the result is still bitwise the host's."""
    rng = np.random.default_rng(n)
    A = ilug.Matrix.from_csr(n, n, *_random_csr(rng, n, density))
    cfg = _ilut_cfg(ilug, 1e-4, lfill)
    _same(ilug.ilu_factorize_device(A, cfg), ilug.ilu_factorize(A, cfg))


@pytest.mark.parametrize("seed", range(4))
def test_device_ilut_random_sparse(ilug, torch_cuda, seed):
    """Unstructured random patterns (fill lands anywhere, long U rows)."""
    rng = np.random.default_rng(100 + seed)
    n = 2000
    A = ilug.Matrix.from_csr(n, n, *_random_csr(rng, n, 0.004))
    for droptol, lfill in ((1e-3, 5), (0.0, 10)):
        cfg = _ilut_cfg(ilug, droptol, lfill)
        _same(ilug.ilu_factorize_device(A, cfg), ilug.ilu_factorize(A, cfg))


@pytest.mark.parametrize("patch", ["error", "replace"])
def test_device_ilut_zero_pivot(ilug, torch_cuda, patch):
    """A zero pivot (structurally absent diagonal at row 3): the same error or
    the same substituted pivot as the host path."""
    n = 6
    rows, cols, vals = [], [], []
    for i in range(n):
        if i > 0:
            rows.append(i), cols.append(i - 1), vals.append(-1.0)
        if i != 3:
            rows.append(i), cols.append(i), vals.append(4.0)
    rp = np.zeros(n + 1, np.int64)
    for r in rows:
        rp[r + 1] += 1
    rp = np.cumsum(rp)
    A = ilug.Matrix.from_csr(n, n, rp, np.array(cols, np.int64), np.array(vals))
    cfg = _ilut_cfg(ilug, 1e-3, 2, patch)
    if patch == "error":
        for fn in (ilug.ilu_factorize, ilug.ilu_factorize_device):
            with pytest.raises(ilug.IlugError) as e:
                fn(A, cfg)
            assert e.value.status == 3 and "step 3" in e.value.message
    else:
        _same(ilug.ilu_factorize_device(A, cfg), ilug.ilu_factorize(A, cfg))


def test_device_ilut_large_bitwise(ilug, torch_cuda):
    """2.1 M rows of the C2 operator family (deep dependency chains): bitwise."""
    A = ilug.Matrix.generate("pressure27(128,128,128)")
    cfg = _ilut_cfg(ilug, 1e-3, 5)
    _same(ilug.ilu_factorize_device(A, cfg), ilug.ilu_factorize(A, cfg))


@pytest.mark.parametrize("quota", ["0", "1", "7", "256"])
def test_device_ilut_row_quota_bitwise(ilug, torch_cuda, monkeypatch, quota):
    """Warps retiring after `quota` rows (fresh CTAs take the next tickets;
    0 = persistent grid) give the same factors: the row order is the ticket
    order either way (kernels/ilut.cu launch_ilut)."""
    monkeypatch.setenv("ILUG_ILUT_QUOTA", quota)
    A = ilug.Matrix.generate("pressure27(20,20,20)")
    cfg = _ilut_cfg(ilug, 1e-3, 5)
    _same(ilug.ilu_factorize_device(A, cfg), ilug.ilu_factorize(A, cfg))


@pytest.mark.parametrize("spec", ["pressure27(20,20,20)", "cutcell(14,14,14)", "stencil27(9,7,5)"])
@pytest.mark.parametrize("droptol,lfill", [(1e-3, 5), (0.0, 40)])
def test_device_ilut_half_warp_rows_bitwise(ilug, torch_cuda, monkeypatch, spec, droptol, lfill):
    """ILUG_ILUT_HALF=1: two rows per warp, one per 16-lane half, 160-entry
    working rows (wider ones take the capacity relaunch): identical factors."""
    monkeypatch.setenv("ILUG_ILUT_HALF", "1")
    A = ilug.Matrix.generate(spec)
    cfg = _ilut_cfg(ilug, droptol, lfill)
    _same(ilug.ilu_factorize_device(A, cfg), ilug.ilu_factorize(A, cfg))


@pytest.mark.parametrize("chunk", ["2", "5"])
def test_device_ilut_chunked_tickets_bitwise(ilug, torch_cuda, monkeypatch, chunk):
    """ILUG_ILUT_CHUNK: consecutive rows per warp ticket (a started chunk is
    finished past the quota): identical factors."""
    monkeypatch.setenv("ILUG_ILUT_CHUNK", chunk)
    monkeypatch.setenv("ILUG_ILUT_QUOTA", "3")
    A = ilug.Matrix.generate("pressure27(20,20,20)")
    cfg = _ilut_cfg(ilug, 1e-3, 5)
    _same(ilug.ilu_factorize_device(A, cfg), ilug.ilu_factorize(A, cfg))
