"""Device AMG setup (kernels/amg_setup.cu): strength,
PMIS, direct and MM-ext interpolation, transposes and the Galerkin products on
the GPU.
Every level's A, P and R must be BITWISE the reference's (src/amg.cpp:18-390),
and the device hierarchy must equal the host setup's at a larger size."""
import numpy as np
import pytest

from conftest import bitwise

pytestmark = pytest.mark.gpu

SPECS = ["poisson3d(16,16,16)", "pressure27(12,12,12)", "cutcell(12,12,12)", "poisson2d(33,31)",
         "anisotropic2d(24,24,0.1)", "stencil27(10,10,10)"]
PMIS = {"amg.coarsening": "pmis", "amg.interpolation": "direct"}


def _same(a, b):
    return (np.array_equal(a[0], b[0]) and np.array_equal(np.asarray(a[1], np.int64), np.asarray(b[1], np.int64))
            and bitwise(np.asarray(a[2]), np.asarray(b[2])))


@pytest.mark.parametrize("spec", SPECS)
@pytest.mark.parametrize("extra", [{}, {"amg.theta": "0.5", "amg.pmis_seed": "7"}, {"amg.coarse_size": "40"},
                                   {"amg.interpolation": "mm_ext"},
                                   {"amg.interpolation": "mm_ext", "amg.theta": "0.5", "amg.pmis_seed": "3"}])
def test_device_setup_bitwise_reference(ilug, ref, torch_cuda, spec, extra):
    kv = dict(PMIS, **extra)
    A = ilug.Matrix.generate(spec)
    H = ilug.Hierarchy(A, ilug.Config().update(dict(kv, **{"device.amg_setup": "device"})), host_only=True)
    Hr = ref.amg(ref.mat(*A.csr()), ref.cfg(kv))
    assert H.levels == ref.amg_levels(Hr)
    for k in range(H.levels):
        for which in ("A", "P", "R") if k + 1 < H.levels else ("A",):
            assert _same(H.level_matrix(k, which).csr(), ref.amg_level(Hr, k, which)), f"level {k} {which}"


@pytest.mark.parametrize("spec", ["pressure27(48,48,48)", "poisson3d(64,64,64)"])
@pytest.mark.parametrize("interp", ["direct", "mm_ext"])
def test_device_setup_equals_host_setup(ilug, torch_cuda, spec, interp):
    kv = dict(PMIS, **{"amg.interpolation": interp})
    A = ilug.Matrix.generate(spec)
    Hd = ilug.Hierarchy(A, ilug.Config().update(dict(kv, **{"device.amg_setup": "device"})), host_only=True)
    Hh = ilug.Hierarchy(A, ilug.Config().update(dict(kv, **{"device.amg_setup": "host"})), host_only=True)
    assert Hd.levels == Hh.levels
    for k in range(Hd.levels):
        for which in ("A", "P", "R") if k + 1 < Hd.levels else ("A",):
            assert _same(Hd.level_matrix(k, which).csr(), Hh.level_matrix(k, which).csr()), f"level {k} {which}"


def test_device_setup_requires_pmis(ilug, torch_cuda):
    A = ilug.Matrix.generate("poisson2d(16,16)")
    with pytest.raises(ilug.IlugError):
        ilug.Hierarchy(A, ilug.Config().update({"device.amg_setup": "device"}), host_only=True)  # rs_greedy


def test_run_solve_device_setup_matches_host_setup(ilug, torch_cuda):
    """run_solve with the GPU setup (auto) and with the host setup: same
    hierarchy, same iterations and the same final residual bits."""
    kv = dict(PMIS, **{"smoother.kind": "ilu", "trisolve.m_lower": "5", "trisolve.m_upper": "5",
                       "krylov.tol": "1e-8"})
    A = ilug.Matrix.generate("pressure27(32,32,32)")
    a = ilug.run_solve(A, ilug.Config().update(dict(kv, **{"device.amg_setup": "auto"})))
    b = ilug.run_solve(A, ilug.Config().update(dict(kv, **{"device.amg_setup": "host"})))
    assert a["iterations"] == b["iterations"] and a["levels"] == b["levels"]
    assert a["final_relres"] == b["final_relres"]
