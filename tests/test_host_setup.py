"""CPU: the native host setup (generators, ILU(0)/ILUT, AMG hierarchy) is
bitwise the reference's on identical inputs — the prerequisite for bitwise
sweeps and V-cycles on the device. Runs without a GPU."""
import numpy as np
import pytest

from conftest import bitwise

SPECS = ["poisson2d(20,17)", "poisson3d(8,9,7)", "pressure27(10,10,10)", "cutcell(12,12,12)",
         "anisotropic2d(16,12,0.001)", "stencil27(6,7,8)"]
ILU = [dict(), {"ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5"},
       {"ilu.variant": "ilut", "ilu.droptol": "1e-2", "ilu.lfill": "1"},
       {"ilu.variant": "ilut", "ilu.droptol": "0", "ilu.lfill": "0"}]


def _same(a, b):
    return all(bitwise(x, y) if x.dtype == np.float64 else np.array_equal(x, y) for x, y in zip(a, b))


@pytest.mark.parametrize("spec", ["poisson1d(10)", "poisson2d(9,7)", "anisotropic2d(8,6,0.01)", "poisson2d(1,5)"])
def test_reference_generators_identical(ilug, ref, spec):
    assert _same(ilug.Matrix.generate(spec).csr(), ref.arrays(ref.generate(spec)))


def test_3d_generators_shape():
    """nnz/structure of the BASELINE generators (SURVEY.md §8a sizes)."""
    import paper_2111_09512_b200 as ilug
    A = ilug.Matrix.generate("poisson3d(64,64,64)")
    assert A.rows == 262144 and A.nnz == 1810432  # C1
    B = ilug.Matrix.generate("stencil27(8,8,8)")
    assert B.nnz == 22 ** 3  # (3m-2)^3 for m = 8
    for spec in ("pressure27(6,5,4)", "cutcell(6,6,6)", "poisson3d(5,6,7)"):
        rp, ci, v = ilug.Matrix.generate(spec).csr()
        n = len(rp) - 1
        M = np.zeros((n, n))
        for i in range(n):
            M[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
        assert np.allclose(M, M.T, rtol=1e-14, atol=0), spec  # symmetric
        d = np.diag(M)
        off = np.abs(M).sum(1) - np.abs(d)
        assert np.all(d >= off * (1 - 1e-12)), spec  # weakly diagonally dominant


@pytest.mark.parametrize("spec", SPECS)
@pytest.mark.parametrize("kv", ILU, ids=lambda d: "-".join(d.values()) or "ilu0")
def test_ilu_factors_bitwise(ilug, ref, spec, kv):
    A = ilug.Matrix.generate(spec)
    L, U = ilug.ilu_factorize(A, ilug.Config().update(kv))
    Lr, Ur, _, _ = ref.factors_arrays(ref.ilu(ref.mat(*A.csr()), ref.cfg(kv)))
    assert _same(L.csr(), Lr)
    assert _same(U.csr(), Ur)


@pytest.mark.parametrize("spec", ["pressure27(40,40,40)", "poisson3d(48,48,48)"])
def test_ilut_pipelined_parallel_bitwise(ilug, ref, spec):
    """Sizes large enough for the pipelined multi-worker ILUT (and level-parallel
    ILU(0)): still bitwise the serial reference."""
    kv = {"ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5"}
    A = ilug.Matrix.generate(spec)
    for cfg in (kv, {}):
        L, U = ilug.ilu_factorize(A, ilug.Config().update(cfg))
        Lr, Ur, _, _ = ref.factors_arrays(ref.ilu(ref.mat(*A.csr()), ref.cfg(cfg)))
        assert _same(L.csr(), Lr) and _same(U.csr(), Ur)


def test_ilu0_zero_pivot_policy(ilug, ref):
    # a_00 = 0 with the diagonal stored: error by default, patched under replace
    rp, ci, v = np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([0.0, 1.0, 1.0, 1.0])
    A = ilug.Matrix.from_csr(2, 2, rp, ci, v)
    with pytest.raises(ilug.IlugError) as e:
        ilug.ilu_factorize(A, ilug.Config())
    assert e.value.status == 3 and "zero pivot at step 0" in e.value.message
    L, U = ilug.ilu_factorize(A, ilug.Config().set("ilu.pivot_patch", "replace"))
    Lr, Ur, _, _ = ref.factors_arrays(ref.ilu(ref.mat(rp, ci, v), ref.cfg({"ilu.pivot_patch": "replace"})))
    assert _same(U.csr(), Ur) and _same(L.csr(), Lr)


def test_ilu0_requires_structural_diagonal(ilug):
    A = ilug.Matrix.from_csr(2, 2, [0, 1, 2], [1, 0], [1.0, 1.0])
    with pytest.raises(ilug.IlugError) as e:
        ilug.ilu_factorize(A, ilug.Config())
    assert e.value.status == 2 and "structurally absent" in e.value.message


AMG = [{}, {"amg.coarsening": "pmis"}, {"amg.coarsening": "pmis", "amg.interpolation": "mm_ext"},
       {"amg.interpolation": "mm_ext"}, {"amg.theta": "0.5", "amg.coarse_size": "40"},
       {"amg.max_levels": "3"}]


@pytest.mark.parametrize("spec", ["poisson2d(32,32)", "anisotropic2d(24,24,0.1)", "poisson3d(12,12,12)",
                                  "pressure27(10,10,10)", "cutcell(12,12,12)"])
@pytest.mark.parametrize("kv", AMG, ids=lambda d: "-".join(d.values()) or "default")
def test_amg_hierarchy_bitwise(ilug, ref, spec, kv):
    A = ilug.Matrix.generate(spec)
    H = ilug.Hierarchy(A, ilug.Config().update(kv), host_only=True)
    Hr = ref.amg(ref.mat(*A.csr()), ref.cfg(kv))
    assert H.levels == ref.amg_levels(Hr)
    for k in range(H.levels):
        for w in ("A", "P", "R") if k + 1 < H.levels else ("A",):
            assert _same(H.level_matrix(k, w).csr(), ref.amg_level(Hr, k, w)), (k, w)
    assert H.operator_complexity == ref.L.ref_amg_operator_complexity(Hr)


def test_hierarchy_host_only_refuses_device_calls(ilug):
    H = ilug.Hierarchy(ilug.Matrix.generate("poisson2d(8,8)"), ilug.Config(), host_only=True)
    with pytest.raises(ilug.IlugError) as e:
        H.vcycle(0, 0)
    assert e.value.status == 2


def test_setup_thread_count_invariance(ilug, monkeypatch):
    """Host setup loops are row-parallel with disjoint outputs: results do not
    depend on the worker count (checked in a subprocess with ILUG_THREADS=1)."""
    import json
    import subprocess
    import sys
    code = (
        "import sys, json, hashlib; sys.path.insert(0, %r);"
        "import paper_2111_09512_b200 as m;"
        "A = m.Matrix.generate('pressure27(14,14,14)');"
        "H = m.Hierarchy(A, m.Config().set('amg.coarsening','pmis'), host_only=True);"
        "L, U = m.ilu_factorize(A, m.Config());"
        "h = hashlib.sha256();"
        "[h.update(a.tobytes()) for k in range(H.levels) for a in H.level_matrix(k,'A').csr()];"
        "[h.update(a.tobytes()) for a in U.csr()];"
        "print(json.dumps(h.hexdigest()))"
    ) % (ilug.__path__[0] + "/..",)
    outs = []
    for t in ("1", "5"):
        env = dict(__import__("os").environ, ILUG_THREADS=t)
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                                   check=True).stdout)
    assert outs[0] == outs[1]
