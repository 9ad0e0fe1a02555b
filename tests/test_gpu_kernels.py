"""GPU parity of the hot-path kernels (K1-K6) against the oracle.

Bar (task spec ③ and SURVEY.md §8): the device and the reference perform the
same fp64 operations in the same order (thread-per-row, ascending columns,
--fmad=false), so the sweeps, scalings, direct solves, SpMVs and smoothers
must be BITWISE equal to oracle/_ref; the unscaled Jacobi form (no reference
function) must agree with the scaled iteration within 1e-12 relative.
"""
import numpy as np
import pytest

from conftest import bitwise, rel_err

pytestmark = pytest.mark.gpu

SPECS = ["poisson3d(16,16,16)", "pressure27(12,12,12)", "cutcell(16,16,16)", "poisson2d(33,31)"]
ILU = [dict(), {"ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5"}]


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _factors(ilug, ref, spec, kv, scaling, direct=False, upper="scaled"):
    A = ilug.Matrix.generate(spec)
    L, U = ilug.ilu_factorize(A, ilug.Config().update(kv))
    f = ilug.Factors.from_csr(A.rows, L.csr(), U.csr(), scaling=scaling, direct=direct, upper=upper)
    Ar = ref.mat(*A.csr())
    fr = ref.scale(ref.ilu(Ar, ref.cfg(kv)), scaling)
    return A, L.csr(), U.csr(), f, fr


@pytest.mark.parametrize("spec", SPECS)
@pytest.mark.parametrize("kv", ILU)
@pytest.mark.parametrize("scaling", ["row", "row_col"])
def test_k1_scaling_bitwise(ilug, ref, torch_cuda, spec, kv, scaling):
    _, _, _, f, fr = _factors(ilug, ref, spec, kv, scaling)
    (rp, ci, v), rs, cs = f.download_upper()
    _, Ur, rsr, csr_ = ref.factors_arrays(fr)
    assert np.array_equal(rp, Ur[0]) and np.array_equal(ci, Ur[1])
    assert bitwise(v, Ur[2])
    assert bitwise(rs, rsr)
    if scaling == "row_col":
        assert bitwise(cs, csr_)
    else:
        assert cs is None and csr_ is None


@pytest.mark.parametrize("spec", SPECS)
@pytest.mark.parametrize("kv", ILU)
@pytest.mark.parametrize("scaling", ["row", "row_col"])
def test_k2_upper_sweeps_bitwise(ilug, ref, torch_cuda, spec, kv, scaling):
    A, _, _, f, fr = _factors(ilug, ref, spec, kv, scaling)
    b = np.random.default_rng(11).uniform(-1, 1, A.rows)
    bd = _dev(torch_cuda, b)
    x = torch_cuda.empty_like(bd)
    for m in (1, 2, 3, 5, 10):
        f.sweep_upper(bd, x, m)
        assert bitwise(_host(x), ref.richardson_upper_scaled(fr, b, m)), f"m={m}"


@pytest.mark.parametrize("spec", SPECS)
@pytest.mark.parametrize("kv", ILU)
def test_k3_lower_sweeps_bitwise(ilug, ref, torch_cuda, spec, kv):
    A, L, _, f, _ = _factors(ilug, ref, spec, kv, "row")
    Lr = ref.mat(*L)
    b = np.random.default_rng(12).uniform(-1, 1, A.rows)
    bd = _dev(torch_cuda, b)
    y = torch_cuda.empty_like(bd)
    for m in (1, 2, 4, 7):
        f.sweep_lower(bd, y, m)
        assert bitwise(_host(y), ref.richardson_lower(Lr, b, m)), f"m={m}"


@pytest.mark.parametrize("spec", SPECS)
def test_k2_jacobi_unscaled_matches_scaled(ilug, ref, port, torch_cuda, spec):
    """a11b(i): x <- D^-1 (b - N x) on the unscaled U is the same iteration as the
    scaled Richardson (1e-12 relative), and bitwise the C restatement."""
    A, _, U, fj, fr = _factors(ilug, ref, spec, {}, "row", upper="jacobi")
    b = np.random.default_rng(13).uniform(-1, 1, A.rows)
    bd = _dev(torch_cuda, b)
    x = torch_cuda.empty_like(bd)
    for m in (1, 3, 6):
        fj.sweep_upper(bd, x, m)
        got = _host(x)
        assert rel_err(got, ref.richardson_upper_scaled(fr, b, m)) < 1e-12
        assert bitwise(got, port.jacobi_upper(U, b, m))


@pytest.mark.parametrize("spec", SPECS)
@pytest.mark.parametrize("scaling", ["none", "row", "row_col"])
def test_k5_direct_solves_bitwise(ilug, ref, torch_cuda, spec, scaling):
    A, L, U, f, fr = _factors(ilug, ref, spec, {}, scaling, direct=True)
    b = np.random.default_rng(14).uniform(-1, 1, A.rows)
    bd = _dev(torch_cuda, b)
    y = torch_cuda.empty_like(bd)
    f.solve_lower(bd, y)
    assert bitwise(_host(y), ref.solve_lower_direct(ref.mat(*L), b))
    f.solve_upper(bd, y)
    want = ref.solve_upper_direct(ref.mat(*U), b) if scaling == "none" else ref.solve_upper_scaled_direct(fr, b)
    assert bitwise(_host(y), want)


@pytest.mark.parametrize("spec", SPECS + ["stencil27(9,10,11)"])
def test_k6_spmv_residual_bitwise(ilug, ref, torch_cuda, spec):
    A = ilug.Matrix.generate(spec)
    D = ilug.DeviceMatrix(A)
    Ar = ref.mat(*A.csr())
    rng = np.random.default_rng(15)
    x, b = rng.uniform(-1, 1, A.rows), rng.uniform(-1, 1, A.rows)
    xd, bd = _dev(torch_cuda, x), _dev(torch_cuda, b)
    y = torch_cuda.empty_like(xd)
    D.spmv(xd, y)
    assert bitwise(_host(y), ref.spmv(Ar, x, A.rows))
    D.residual(xd, bd, y)
    assert bitwise(_host(y), ref.residual(Ar, x, b))


SMOOTHERS = [
    {"smoother.kind": "ilu", "trisolve.m_lower": 5, "trisolve.m_upper": 5},
    {"smoother.kind": "ilu", "trisolve.m_lower": 1, "trisolve.m_upper": 1},
    {"smoother.kind": "ilu", "trisolve.m_lower": 3, "trisolve.m_upper": 2, "scaling": "row_col"},
    {"smoother.kind": "ilu", "trisolve.mode": "direct"},
    {"smoother.kind": "ilu", "trisolve.mode": "direct", "scaling": "none"},
    {"smoother.kind": "ilu", "ilu.variant": "ilut", "trisolve.m_lower": 4, "trisolve.m_upper": 4},
    {"smoother.kind": "gauss_seidel"},
    {"smoother.kind": "jacobi", "smoother.sweeps": 3},
    {"smoother.kind": "l1_jacobi"},
    {"smoother.kind": "poly_gs", "smoother.poly_degree": 3},
]


@pytest.mark.parametrize("spec", ["poisson3d(14,13,12)", "pressure27(10,10,10)", "cutcell(14,14,14)"])
@pytest.mark.parametrize("kv", SMOOTHERS, ids=lambda d: "-".join(f"{v}" for v in d.values()))
def test_k4_smoother_bitwise(ilug, ref, torch_cuda, spec, kv):
    A = ilug.Matrix.generate(spec)
    cfg = ilug.Config().update(kv)
    S = ilug.Smoother(A, cfg)
    Ar = ref.mat(*A.csr())
    Sr = ref.smoother(Ar, ref.cfg(kv))
    rng = np.random.default_rng(16)
    b, x0 = rng.uniform(-1, 1, A.rows), rng.uniform(-1, 1, A.rows)
    xd = _dev(torch_cuda, x0)
    nrm = S.smooth(_dev(torch_cuda, b), xd, want_norm=True)
    want, want_nrm = ref.smooth(Ar, Sr, b, x0)
    assert bitwise(_host(xd), want)
    assert abs(nrm - want_nrm) <= 1e-12 * max(1.0, want_nrm)


def test_k4_ilu_sweep_fixed_point(ilug, torch_cuda):
    """Every smoother leaves the exact solution fixed (tests/test_smoother.cpp:37-49)."""
    A = ilug.Matrix.generate("poisson3d(10,10,10)")
    D = ilug.DeviceMatrix(A)
    xs = np.random.default_rng(5).uniform(-1, 1, A.rows)
    xd = _dev(torch_cuda, xs)
    bd = torch_cuda.empty_like(xd)
    D.spmv(xd, bd)
    for kv in SMOOTHERS:
        S = ilug.Smoother(A, ilug.Config().update(kv))
        x = xd.clone()
        S.smooth(bd, x)
        assert rel_err(_host(x), xs) < 1e-13, kv


def test_c1_poisson64_sweeps(ilug, ref, torch_cuda):
    """C1: 7-point 64^3, ILU(0), row-scaled U, 5 sweeps vs the reference (bitwise),
    unscaled Jacobi within 1e-12, and both approach the direct solve."""
    A, L, U, f, fr = _factors(ilug, ref, "poisson3d(64,64,64)", {}, "row", direct=True)
    fj = ilug.Factors.from_csr(A.rows, L, U, scaling="row", upper="jacobi")
    b = np.random.default_rng(42).uniform(-1, 1, A.rows)
    bd = _dev(torch_cuda, b)
    x = torch_cuda.empty_like(bd)
    f.sweep_upper(bd, x, 5)
    xs = _host(x)
    assert bitwise(xs, ref.richardson_upper_scaled(fr, b, 5))
    fj.sweep_upper(bd, x, 5)
    assert rel_err(_host(x), xs) < 1e-12
    f.solve_upper(bd, x)
    xd = _host(x)
    assert bitwise(xd, ref.solve_upper_scaled_direct(fr, b))
    assert rel_err(xs, xd) < 5e-2  # truncated Neumann series, m = 5


def test_c3_cutcell_scaled_vs_unscaled(ilug, ref, port, torch_cuda):
    """C3: coefficient jumps over ~16 orders of magnitude. Row scaling collapses
    dep(U); scaled and unscaled-Jacobi sweeps agree to 1e-12; plain Richardson on
    the unscaled factor diverges (the paper's motivating failure)."""
    A, L, U, f, fr = _factors(ilug, ref, "cutcell(32,32,32)", {}, "row", direct=True)
    Ur = ref.mat(*U)
    dep_u = ref.departure(Ur, 2)
    (rp, ci, v), _, _ = f.download_upper()
    dep_s = port.departure((rp, ci, v))
    assert dep_u > 1e6 * dep_s, (dep_u, dep_s)
    fj = ilug.Factors.from_csr(A.rows, L, U, scaling="row", upper="jacobi")
    b = np.random.default_rng(3).uniform(-1, 1, A.rows)
    bd = _dev(torch_cuda, b)
    x = torch_cuda.empty_like(bd)
    f.solve_upper(bd, x)
    direct = _host(x)
    errs = []
    for m in (5, 20, 40):
        f.sweep_upper(bd, x, m)
        xs = _host(x)
        assert bitwise(xs, ref.richardson_upper_scaled(fr, b, m))
        fj.sweep_upper(bd, x, m)
        assert rel_err(_host(x), xs) < 1e-12
        errs.append(rel_err(xs, direct))
    assert errs[0] > errs[1] > errs[2]


@pytest.mark.parametrize("schedule", ["cta", "cta1", "flags", "vflags"])
@pytest.mark.parametrize("spec,kv", [("poisson3d(24,24,20)", {}),
                                     ("pressure27(16,16,16)", {"ilu.variant": "ilut", "ilu.droptol": "1e-3",
                                                               "ilu.lfill": "5"})])
def test_k5_both_schedules_bitwise(ilug, ref, torch_cuda, monkeypatch, schedule, spec, kv):
    """Every level-set schedule (cluster-synchronous, single CTA, sync-free
    separate flags, sync-free value flags) gives the serial result bitwise, for
    the triangular solves and the Gauss-Seidel sweep."""
    monkeypatch.setenv("ILUG_LEVELSET", schedule)
    A, L, U, f, fr = _factors(ilug, ref, spec, kv, "row", direct=True)
    b = np.random.default_rng(31).uniform(-1, 1, A.rows)
    bd = _dev(torch_cuda, b)
    y = torch_cuda.empty_like(bd)
    f.solve_lower(bd, y)
    assert bitwise(_host(y), ref.solve_lower_direct(ref.mat(*L), b))
    f.solve_upper(bd, y)
    assert bitwise(_host(y), ref.solve_upper_scaled_direct(fr, b))
    S = ilug.Smoother(A, ilug.Config().set("smoother.kind", "gauss_seidel"))
    x0 = np.random.default_rng(32).uniform(-1, 1, A.rows)
    xd = _dev(torch_cuda, x0)
    S.smooth(bd, xd)
    Ar = ref.mat(*A.csr())
    want, _ = ref.smooth(Ar, ref.smoother(Ar, ref.cfg({"smoother.kind": "gauss_seidel"})), b, x0)
    assert bitwise(_host(xd), want)


VF_FORMS = ["0", "1", "2", "4", "8", "83", "16", "88", "164", "168", "324"]


@pytest.mark.parametrize("sub", VF_FORMS)
@pytest.mark.parametrize("spec,kv", [("poisson3d(40,40,30)", {}),
                                     ("pressure27(24,24,20)", {"ilu.variant": "ilut", "ilu.droptol": "1e-3",
                                                               "ilu.lfill": "5"})])
def test_k5_value_flag_forms_bitwise(ilug, ref, torch_cuda, monkeypatch, sub, spec, kv):
    """Every form of the sync-free value-flag kernel (thread per row with 16- or
    8-entry chunks; 2/4/8/16 lanes per row with the ordered shuffle chain) gives
    the serial solves and the GS sweep bitwise."""
    monkeypatch.setenv("ILUG_LEVELSET", "vflags")
    monkeypatch.setenv("ILUG_VF_SUB", sub)
    A, L, U, f, fr = _factors(ilug, ref, spec, kv, "row", direct=True)
    b = np.random.default_rng(37).uniform(-1, 1, A.rows)
    bd = _dev(torch_cuda, b)
    y = torch_cuda.empty_like(bd)
    for _ in range(2):
        f.solve_lower(bd, y)
        assert bitwise(_host(y), ref.solve_lower_direct(ref.mat(*L), b))
        f.solve_upper(bd, y)
        assert bitwise(_host(y), ref.solve_upper_scaled_direct(fr, b))
    S = ilug.Smoother(A, ilug.Config().set("smoother.kind", "gauss_seidel"))
    x0 = np.random.default_rng(38).uniform(-1, 1, A.rows)
    xd = _dev(torch_cuda, x0)
    S.smooth(bd, xd)
    Ar = ref.mat(*A.csr())
    want, _ = ref.smooth(Ar, ref.smoother(Ar, ref.cfg({"smoother.kind": "gauss_seidel"})), b, x0)
    assert bitwise(_host(xd), want)


@pytest.mark.parametrize("sub", [""] + VF_FORMS)
def test_k5_long_rows_gs_bitwise(ilug, ref, torch_cuda, monkeypatch, sub):
    """Gauss-Seidel on coarse AMG operators (rows of 40-110 entries: several
    32-entry passes for the narrow forms, one pass for the 64/128-entry
    forms the default picks there) bitwise the reference's sweep."""
    monkeypatch.setenv("ILUG_LEVELSET", "vflags")
    if sub:
        monkeypatch.setenv("ILUG_VF_SUB", sub)
    A = ilug.Matrix.generate("pressure27(40,40,40)")
    H = ilug.Hierarchy(A, ilug.Config().update({"amg.coarsening": "pmis"}), host_only=True)
    widths = []
    for lvl in range(1, min(H.levels - 1, 5)):
        M = H.level_matrix(lvl, "A")
        rp, ci, v = M.csr()
        widths.append(int(np.diff(rp).max()))
        b = np.random.default_rng(40 + lvl).uniform(-1, 1, M.rows)
        x0 = np.random.default_rng(50 + lvl).uniform(-1, 1, M.rows)
        S = ilug.Smoother(M, ilug.Config().update({"smoother.kind": "gauss_seidel", "smoother.sweeps": "2"}))
        xd = _dev(torch_cuda, x0)
        S.smooth(_dev(torch_cuda, b), xd)
        Mr = ref.mat(rp, ci, v)
        want, _ = ref.smooth(Mr, ref.smoother(Mr, ref.cfg({"smoother.kind": "gauss_seidel",
                                                           "smoother.sweeps": "2"})), b, x0)
        assert bitwise(_host(xd), want), f"level {lvl}"
    assert max(widths) > 64


@pytest.mark.parametrize("schedule", ["", "cta", "flags", "vflags"])
def test_k5_wide_dag_bitwise(ilug, ref, torch_cuda, monkeypatch, schedule):
    """A wide DAG (n / levels > 2048: levels wider than a cluster's threads,
    so cluster threads take several rows per level)."""
    if schedule:
        monkeypatch.setenv("ILUG_LEVELSET", schedule)
    A, L, U, f, fr = _factors(ilug, ref, "poisson3d(160,160,40)", {}, "row", direct=True)
    st = f.stats()
    assert A.rows / st["levels_L"] > 2048
    b = np.random.default_rng(33).uniform(-1, 1, A.rows)
    bd = _dev(torch_cuda, b)
    y = torch_cuda.empty_like(bd)
    for _ in range(2):  # epoch-stamped flags: repeated solves need no reset
        f.solve_lower(bd, y)
        assert bitwise(_host(y), ref.solve_lower_direct(ref.mat(*L), b))
        f.solve_upper(bd, y)
        assert bitwise(_host(y), ref.solve_upper_scaled_direct(fr, b))


def test_k5_direct_at_scale_bitwise(ilug, ref, torch_cuda):
    """27-point 128^3 (2.1M rows, sync-free schedule): direct solves bitwise vs
    the reference, and the triangular residual at rounding level."""
    A, L, U, f, fr = _factors(ilug, ref, "pressure27(128,128,128)", {}, "row", direct=True)
    st = f.stats()
    assert A.rows / st["levels_U"] > 2048
    b = np.random.default_rng(34).uniform(-1, 1, A.rows)
    bd = _dev(torch_cuda, b)
    y = torch_cuda.empty_like(bd)
    f.solve_upper(bd, y)
    got = _host(y)
    assert bitwise(got, ref.solve_upper_scaled_direct(fr, b))
    f.solve_lower(bd, y)
    assert bitwise(_host(y), ref.solve_lower_direct(ref.mat(*L), b))


@pytest.mark.parametrize("schedule", ["", "cta", "flags", "vflags"])
def test_k5_deep_chain_bitwise(ilug, ref, torch_cuda, monkeypatch, schedule):
    """A 1D chain (7000 levels of one row: more levels than the warp-per-row
    cluster kernel keeps in shared memory, so the default takes the one-CTA
    kernel): direct solves and the Gauss-Seidel sweep stay bitwise."""
    if schedule:
        monkeypatch.setenv("ILUG_LEVELSET", schedule)
    A, L, U, f, fr = _factors(ilug, ref, "poisson1d(7000)", {}, "row", direct=True)
    assert f.stats()["levels_L"] == 7000
    b = np.random.default_rng(35).uniform(-1, 1, A.rows)
    bd = _dev(torch_cuda, b)
    y = torch_cuda.empty_like(bd)
    f.solve_lower(bd, y)
    assert bitwise(_host(y), ref.solve_lower_direct(ref.mat(*L), b))
    f.solve_upper(bd, y)
    assert bitwise(_host(y), ref.solve_upper_scaled_direct(fr, b))
    S = ilug.Smoother(A, ilug.Config().set("smoother.kind", "gauss_seidel"))
    x0 = np.random.default_rng(36).uniform(-1, 1, A.rows)
    xd = _dev(torch_cuda, x0)
    S.smooth(bd, xd)
    Ar = ref.mat(*A.csr())
    want, _ = ref.smooth(Ar, ref.smoother(Ar, ref.cfg({"smoother.kind": "gauss_seidel"})), b, x0)
    assert bitwise(_host(xd), want)


def test_direct_cusparse_comparison_path(ilug, ref, torch_cuda, monkeypatch):
    """ILUG_DIRECT=cusparse (the library comparison point for K5): the same
    solves through cuSPARSE SpSV agree with the bitwise K5 result to rounding,
    and a direct-mode GMRES+AMG solve through it converges in the same number
    of iterations (+-1)."""
    A, L, U, f, fr = _factors(ilug, ref, "pressure27(24,24,24)", {"ilu.variant": "ilut", "ilu.droptol": "1e-3",
                                                                  "ilu.lfill": "5"}, "row", direct=True)
    b = np.random.default_rng(41).uniform(-1, 1, A.rows)
    bd = _dev(torch_cuda, b)
    y = torch_cuda.empty_like(bd)
    f.solve_lower(bd, y)
    yl = _host(y)
    f.solve_upper(bd, y)
    yu = _host(y)
    monkeypatch.setenv("ILUG_DIRECT", "cusparse")
    g = ilug.Factors.from_csr(A.rows, L, U, scaling="row", direct=True)
    g.solve_lower(bd, y)
    assert rel_err(_host(y), yl) < 1e-12
    g.solve_upper(bd, y)
    assert rel_err(_host(y), yu) < 1e-12
    kv = {"smoother.kind": "ilu", "ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5",
          "trisolve.mode": "direct", "amg.coarsening": "pmis", "krylov.tol": "1e-8"}
    got = ilug.run_solve(A, ilug.Config().update(kv))
    monkeypatch.delenv("ILUG_DIRECT")
    want = ilug.run_solve(A, ilug.Config().update(kv))
    assert got["converged"] == "true" and abs(int(got["iterations"]) - int(want["iterations"])) <= 1


@pytest.mark.parametrize("scaling,upper,direct", [("row", "scaled", True), ("row_col", "scaled", False),
                                                  ("none", "jacobi", True)])
def test_ilu0_refactor_bitwise(ilug, ref, torch_cuda, scaling, upper, direct):
    """Numeric refactorisation with the same pattern (new coefficients, seed 7):
    sweeps and direct solves bitwise those of factors built from scratch."""
    A1 = ilug.Matrix.generate("pressure27(20,18,16,2111)")
    A2 = ilug.Matrix.generate("pressure27(20,18,16,7)")
    assert np.array_equal(A1.csr()[1], A2.csr()[1])
    cfg = ilug.Config()
    f = ilug.Factors.create(A1, cfg, scaling=scaling, upper=upper, direct=direct)
    f.refactor(A2)
    g = ilug.Factors.create(A2, cfg, scaling=scaling, upper=upper, direct=direct)
    b = np.random.default_rng(51).uniform(-1, 1, A2.rows)
    bd = _dev(torch_cuda, b)
    y1, y2 = torch_cuda.empty_like(bd), torch_cuda.empty_like(bd)
    for m in (1, 3, 6):
        f.sweep_lower(bd, y1, m), g.sweep_lower(bd, y2, m)
        assert bitwise(_host(y1), _host(y2))
        f.sweep_upper(bd, y1, m), g.sweep_upper(bd, y2, m)
        assert bitwise(_host(y1), _host(y2))
    if direct:
        f.solve_lower(bd, y1), g.solve_lower(bd, y2)
        assert bitwise(_host(y1), _host(y2))
        f.solve_upper(bd, y1), g.solve_upper(bd, y2)
        assert bitwise(_host(y1), _host(y2))
    f.refactor(A1)  # and back: the symbolic data are reused
    h = ilug.Factors.create(A1, cfg, scaling=scaling, upper=upper, direct=direct)
    f.sweep_upper(bd, y1, 4), h.sweep_upper(bd, y2, 4)
    assert bitwise(_host(y1), _host(y2))


def test_ilu0_refactor_rejects_other_patterns(ilug, torch_cuda):
    f = ilug.Factors.create(ilug.Matrix.generate("pressure27(10,10,10)"), ilug.Config())
    with pytest.raises(ilug.IlugError) as e:
        f.refactor(ilug.Matrix.generate("poisson3d(10,10,10)"))
    assert e.value.status == 2 and "pattern" in e.value.message
    t = ilug.Factors.create(ilug.Matrix.generate("pressure27(10,10,10)"),
                            ilug.Config().update({"ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5"}))
    with pytest.raises(ilug.IlugError) as e:
        t.refactor(ilug.Matrix.generate("pressure27(10,10,10)"))
    assert e.value.status == 2


def _random_dominant(ilug, n, per_row, seed):
    """Unstructured diagonally dominant matrix: far more than 255 distinct
    column offsets (the SELL-D8 coding must decline it)."""
    rng = np.random.default_rng(seed)
    cols = np.concatenate([np.arange(n)[:, None], rng.integers(0, n, (n, per_row))], axis=1)
    cols.sort(axis=1)
    keep = np.ones_like(cols, dtype=bool)
    keep[:, 1:] = cols[:, 1:] != cols[:, :-1]
    vals = rng.uniform(-1, 1, cols.shape)
    vals[cols == np.arange(n)[:, None]] = per_row + 2.0
    rp = np.concatenate([[0], np.cumsum(keep.sum(axis=1))])
    return ilug.Matrix.from_csr(n, n, rp, cols[keep], vals[keep])


@pytest.mark.parametrize("which", ["pressure27", "poisson3d", "random"])
def test_sell_d8_coded_columns_bitwise(ilug, ref, torch_cuda, monkeypatch, which):
    """SELL-D8 (1-byte dictionary-coded columns, col = row + offtab[code]) and
    the int32 column stream give the same smoother step bit for bit, and both
    the reference's ilu_smooth_sweep; an unstructured matrix (> 255 offsets)
    stays on the int32 stream."""
    torch = torch_cuda
    if which == "random":
        A = _random_dominant(ilug, 70000, 8, 5)
    else:  # > 65536 rows: the thread-per-row sweep kernel (smaller operators take a warp per row)
        A = ilug.Matrix.generate({"pressure27": "pressure27(48,48,32)", "poisson3d": "poisson3d(50,50,30)"}[which])
    kv = {"smoother.kind": "ilu", "ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5",
          "trisolve.m_lower": "5", "trisolve.m_upper": "5", "smoother.sweeps": "1"}
    b = np.random.default_rng(61).uniform(-1, 1, A.rows)
    x0 = np.random.default_rng(62).uniform(-1, 1, A.rows)
    got = {}
    for d8 in ("1", "0"):
        monkeypatch.setenv("ILUG_SELL_D8", d8)
        S = ilug.Smoother(A, ilug.Config().update(kv))
        xd = _dev(torch, x0)
        S.ilu_sweep(_dev(torch, b), xd)
        got[d8] = _host(xd)
        y = torch.empty(A.rows, dtype=torch.float64, device="cuda")
        DM = ilug.DeviceMatrix(A)
        DM.spmv(_dev(torch, x0), y)
        got[d8 + "spmv"] = _host(y)
    assert bitwise(got["1"], got["0"]) and bitwise(got["1spmv"], got["0spmv"])
    Ar = ref.mat(*A.csr())
    want = ref.ilu_smooth_sweep(Ar, ref.smoother(Ar, ref.cfg(kv)), b, x0)
    assert bitwise(got["1"], want)
    assert bitwise(got["1spmv"], ref.spmv(Ar, x0, A.rows))


@pytest.mark.parametrize("which", ["pressure27", "poisson3d", "random"])
def test_sell_device_layout_matches_host_layout(ilug, ref, torch_cuda, monkeypatch, which):
    """The SELL-C-sigma layout computed on the GPU (row lengths, per-window
    stable sort, the 3 % padding rule, slice offsets) equals the host layout:
    same stored/padded entry counts, same smoother and SpMV bits, both the
    reference's."""
    torch = torch_cuda
    if which == "random":
        A = _random_dominant(ilug, 70000, 8, 7)
    else:
        A = ilug.Matrix.generate({"pressure27": "pressure27(48,48,32)", "poisson3d": "poisson3d(50,50,30)"}[which])
    kv = {"smoother.kind": "ilu", "ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5",
          "trisolve.m_lower": "5", "trisolve.m_upper": "5", "smoother.sweeps": "1"}
    b = np.random.default_rng(71).uniform(-1, 1, A.rows)
    x0 = np.random.default_rng(72).uniform(-1, 1, A.rows)
    got, stats = {}, {}
    for dev in ("1", "0"):
        monkeypatch.setenv("ILUG_SELL_DEVICE_LAYOUT", dev)
        S = ilug.Smoother(A, ilug.Config().update(kv))
        F = ilug.Factors.create(A, ilug.Config().update(kv), scaling="row")
        stats[dev] = F.stats()
        xd = _dev(torch, x0)
        S.ilu_sweep(_dev(torch, b), xd)
        got[dev] = _host(xd)
        y = torch.empty(A.rows, dtype=torch.float64, device="cuda")
        ilug.DeviceMatrix(A).spmv(_dev(torch, x0), y)
        got[dev + "spmv"] = _host(y)
    assert stats["1"] == stats["0"]
    assert bitwise(got["1"], got["0"]) and bitwise(got["1spmv"], got["0spmv"])
    Ar = ref.mat(*A.csr())
    assert bitwise(got["1"], ref.ilu_smooth_sweep(Ar, ref.smoother(Ar, ref.cfg(kv)), b, x0))


@pytest.mark.parametrize("dsm", ["1", "0"])
@pytest.mark.parametrize("spec,kv", [("poisson3d(40,40,30)", {}),
                                     ("pressure27(24,24,20)", {"ilu.variant": "ilut", "ilu.droptol": "1e-3",
                                                               "ilu.lfill": "5"})])
def test_k5_cluster_dsmem_form_bitwise(ilug, ref, torch_cuda, monkeypatch, dsm, spec, kv):
    """The thread-block-cluster form of the value-flag schedule (the solution
    in the clusters' distributed shared memory; forced everywhere it fits with
    ILUG_LEVELSET_DSM=1) and the global form give the serial L / U solves and
    the GS sweep bitwise, repeatedly."""
    monkeypatch.setenv("ILUG_LEVELSET", "vflags")
    monkeypatch.setenv("ILUG_LEVELSET_DSM", dsm)
    A, L, U, f, fr = _factors(ilug, ref, spec, kv, "row", direct=True)
    b = np.random.default_rng(83).uniform(-1, 1, A.rows)
    bd = _dev(torch_cuda, b)
    y = torch_cuda.empty_like(bd)
    for _ in range(2):
        f.solve_lower(bd, y)
        assert bitwise(_host(y), ref.solve_lower_direct(ref.mat(*L), b))
        f.solve_upper(bd, y)
        assert bitwise(_host(y), ref.solve_upper_scaled_direct(fr, b))
    S = ilug.Smoother(A, ilug.Config().update({"smoother.kind": "gauss_seidel", "smoother.sweeps": "2"}))
    x0 = np.random.default_rng(84).uniform(-1, 1, A.rows)
    xd = _dev(torch_cuda, x0)
    S.smooth(bd, xd)
    Ar = ref.mat(*A.csr())
    want, _ = ref.smooth(Ar, ref.smoother(Ar, ref.cfg({"smoother.kind": "gauss_seidel",
                                                       "smoother.sweeps": "2"})), b, x0)
    assert bitwise(_host(xd), want)
