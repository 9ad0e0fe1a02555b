"""GPU parity of the wavefront (temporally blocked) sweeps, kernels/wavefront.cu.

m-1 Richardson/Jacobi sweeps in ONE launch must be BITWISE the per-sweep
kernels and hence the reference (src/trisolve.cpp:94-147, src/smoother.cpp:143-159):
each row is still one thread summing its columns in ascending order, the
fusion only changes when (not how) a row is computed. The path is opt-in
(ILUG_WAVEFRONT=1; measured slower than separate sweeps on B200, see
kernels/wavefront.cu), forced here on matrices small enough for the oracle and
at 96^3.
"""
import numpy as np
import pytest

from conftest import bitwise, rel_err

pytestmark = pytest.mark.gpu

SPECS = ["poisson3d(16,16,16)", "pressure27(12,12,12)", "cutcell(16,16,16)", "poisson2d(33,31)",
         "poisson3d(7,5,3)"]  # the last: one partial tile
ILUT = {"ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5"}


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


@pytest.fixture
def wave_on(monkeypatch):
    monkeypatch.setenv("ILUG_WAVEFRONT", "1")


def _tiles(n):
    return ((n + 31) // 32 * 32 + 127) // 128  # 128-row tiles of the SELL rows


def _factors(ilug, ref, spec, kv, scaling, upper="scaled"):
    A = ilug.Matrix.generate(spec)
    L, U = ilug.ilu_factorize(A, ilug.Config().update(kv))
    f = ilug.Factors.from_csr(A.rows, L.csr(), U.csr(), scaling=scaling, upper=upper)
    fr = ref.scale(ref.ilu(ref.mat(*A.csr()), ref.cfg(kv)), scaling)
    return A, L.csr(), U.csr(), f, fr


@pytest.mark.parametrize("spec", SPECS)
@pytest.mark.parametrize("kv", [{}, ILUT], ids=["ilu0", "ilut"])
@pytest.mark.parametrize("scaling", ["row", "row_col"])
def test_wave_upper_sweeps_bitwise(ilug, ref, torch_cuda, wave_on, spec, kv, scaling):
    A, _, _, f, fr = _factors(ilug, ref, spec, kv, scaling)
    w = f.wave()
    assert w["tiles_U"] == _tiles(A.rows) and w["tiles_L"] == w["tiles_U"]
    b = np.random.default_rng(21).uniform(-1, 1, A.rows)
    bd = _dev(torch_cuda, b)
    x = torch_cuda.empty_like(bd)
    for m in (3, 4, 6, 10):  # 2..9 fused sweeps
        f.sweep_upper(bd, x, m)
        assert bitwise(_host(x), ref.richardson_upper_scaled(fr, b, m)), f"m={m}"
    assert not f.wave()["stalled"]


@pytest.mark.parametrize("spec", SPECS)
@pytest.mark.parametrize("kv", [{}, ILUT], ids=["ilu0", "ilut"])
def test_wave_lower_sweeps_bitwise(ilug, ref, torch_cuda, wave_on, spec, kv):
    A, L, _, f, _ = _factors(ilug, ref, spec, kv, "row")
    Lr = ref.mat(*L)
    b = np.random.default_rng(22).uniform(-1, 1, A.rows)
    bd = _dev(torch_cuda, b)
    y = torch_cuda.empty_like(bd)
    for m in (3, 5, 10, 11):  # 11: beyond the fused limit, per-sweep path
        f.sweep_lower(bd, y, m)
        assert bitwise(_host(y), ref.richardson_lower(Lr, b, m)), f"m={m}"
    assert not f.wave()["stalled"]


@pytest.mark.parametrize("spec", SPECS[:3])
def test_wave_jacobi_upper_bitwise_port(ilug, ref, port, torch_cuda, wave_on, spec):
    A, _, U, fj, fr = _factors(ilug, ref, spec, {}, "row", upper="jacobi")
    assert fj.wave()["tiles_U"] > 0
    b = np.random.default_rng(23).uniform(-1, 1, A.rows)
    bd = _dev(torch_cuda, b)
    x = torch_cuda.empty_like(bd)
    for m in (3, 6):
        fj.sweep_upper(bd, x, m)
        got = _host(x)
        assert bitwise(got, port.jacobi_upper(U, b, m))
        assert rel_err(got, ref.richardson_upper_scaled(fr, b, m)) < 1e-12


SMOOTHERS = [
    {"smoother.kind": "ilu", "trisolve.m_lower": 5, "trisolve.m_upper": 5},
    {"smoother.kind": "ilu", "trisolve.m_lower": 3, "trisolve.m_upper": 2, "scaling": "row_col"},
    {"smoother.kind": "ilu", "trisolve.m_lower": 2, "trisolve.m_upper": 7, "scaling": "row_col"},
    {"smoother.kind": "ilu", "trisolve.m_lower": 4, "trisolve.m_upper": 3, "trisolve.upper": "jacobi"},
    {"smoother.kind": "ilu", "ilu.variant": "ilut", "trisolve.m_lower": 4, "trisolve.m_upper": 4,
     "smoother.sweeps": 2},
]


@pytest.mark.parametrize("spec", ["poisson3d(14,13,12)", "pressure27(10,10,10)", "cutcell(14,14,14)"])
@pytest.mark.parametrize("kv", SMOOTHERS, ids=lambda d: "-".join(f"{v}" for v in d.values()))
def test_wave_smoother_bitwise(ilug, ref, port, torch_cuda, wave_on, spec, kv):
    A = ilug.Matrix.generate(spec)
    S = ilug.Smoother(A, ilug.Config().update(kv))
    rng = np.random.default_rng(24)
    b, x0 = rng.uniform(-1, 1, A.rows), rng.uniform(-1, 1, A.rows)
    xd = _dev(torch_cuda, x0)
    S.smooth(_dev(torch_cuda, b), xd)
    got = _host(xd)
    if kv.get("trisolve.upper") == "jacobi":
        # no reference function for the Jacobi form: compare with the unfused device path
        import os
        os.environ["ILUG_WAVEFRONT"] = "0"
        S0 = ilug.Smoother(A, ilug.Config().update(kv))
        os.environ["ILUG_WAVEFRONT"] = "1"
        assert S0.wave()["tiles_U"] == 0
        x1 = _dev(torch_cuda, x0)
        S0.smooth(_dev(torch_cuda, b), x1)
        assert bitwise(got, _host(x1))
    else:
        Ar = ref.mat(*A.csr())
        want, _ = ref.smooth(Ar, ref.smoother(Ar, ref.cfg(kv)), b, x0)
        assert bitwise(got, want)
    w = S.wave()
    assert w["tiles_U"] > 0 and not w["stalled"]


@pytest.mark.parametrize("env", [{"ILUG_WAVE_CTAS_PER_SM": "1"}, {"ILUG_WAVE_CTAS_PER_SM": "16"},
                                 {"ILUG_WAVE_L2_MB": "1"}, {"ILUG_WAVE_HINTS": "1"},
                                 {"ILUG_SELL_SIGMA": "64"}, {"ILUG_SELL_SIGMA": "1"}, {"ILUG_SELL_SIGMA": "3000"}])
def test_wave_schedules_bitwise(ilug, ref, torch_cuda, wave_on, monkeypatch, env):
    """Grid size (so the lag between sweeps) and the SELL sorting window change
    the schedule, never the result."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    A, L, _, f, fr = _factors(ilug, ref, "pressure27(24,24,24)", {}, "row_col")
    b = np.random.default_rng(25).uniform(-1, 1, A.rows)
    bd = _dev(torch_cuda, b)
    x = torch_cuda.empty_like(bd)
    f.sweep_upper(bd, x, 8)
    assert bitwise(_host(x), ref.richardson_upper_scaled(fr, b, 8))
    f.sweep_lower(bd, x, 8)
    assert bitwise(_host(x), ref.richardson_lower(ref.mat(*L), b, 8))
    assert not f.wave()["stalled"]


@pytest.mark.parametrize("setting", [None, "0"])
def test_wave_off_by_default(ilug, torch_cuda, monkeypatch, setting):
    if setting is None:
        monkeypatch.delenv("ILUG_WAVEFRONT", raising=False)
    else:
        monkeypatch.setenv("ILUG_WAVEFRONT", setting)
    A = ilug.Matrix.generate("poisson3d(70,70,70)")
    L, U = ilug.ilu_factorize(A, ilug.Config())
    f = ilug.Factors.from_csr(A.rows, L.csr(), U.csr(), scaling="row")
    assert f.wave()["tiles_U"] == 0 and f.wave()["tiles_L"] == 0


def test_wave_at_scale_bitwise(ilug, ref, torch_cuda, wave_on):
    """96^3 (885k rows, 6912 tiles, default grid/L2 budget): sweeps bitwise vs
    the reference; repeated launches reuse the epoch-stamped flags."""
    A, L, _, f, fr = _factors(ilug, ref, "poisson3d(96,96,96)", {}, "row")
    assert f.wave()["tiles_U"] == _tiles(A.rows)
    b = np.random.default_rng(26).uniform(-1, 1, A.rows)
    bd = _dev(torch_cuda, b)
    x = torch_cuda.empty_like(bd)
    want = ref.richardson_upper_scaled(fr, b, 5)
    for _ in range(3):
        f.sweep_upper(bd, x, 5)
        assert bitwise(_host(x), want)
    f.sweep_lower(bd, x, 5)
    assert bitwise(_host(x), ref.richardson_lower(ref.mat(*L), b, 5))
    assert not f.wave()["stalled"]


def test_wave_sweeps_fused_entry(ilug, ref, torch_cuda, wave_on):
    """ilug_smoother_sweeps_fused (the bench's per-kernel entry) = nsweeps bare sweeps."""
    A = ilug.Matrix.generate("poisson3d(20,20,20)")
    S = ilug.Smoother(A, ilug.Config().update({"smoother.kind": "ilu"}))
    rng = np.random.default_rng(27)
    x0, rhs = _dev(torch_cuda, rng.uniform(-1, 1, A.rows)), _dev(torch_cuda, rng.uniform(-1, 1, A.rows))
    for which in (0, 1):
        out = torch_cuda.empty_like(x0)
        tmp = torch_cuda.empty(3 * A.rows, dtype=torch_cuda.float64, device="cuda")
        S.sweeps_fused(which, 4, x0, rhs, tmp, out)
        cur = x0.clone()
        nxt = torch_cuda.empty_like(x0)
        for _ in range(4):
            ilug.lib.ilug_smoother_sweep_once(S.h, which, ilug._ptr(cur), ilug._ptr(rhs), ilug._ptr(nxt), None)
            cur, nxt = nxt, cur
        assert bitwise(_host(out), _host(cur))
