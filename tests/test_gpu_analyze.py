"""GPU: iluamg_run_analyze (factor diagnostics of the drop-in ABI) reports the
reference's numbers bitwise — departures from normality of L, U and the row /
row-col scaled U (K1 on the device), Hager condition estimates (K5 solves on
the device, host reductions in the reference order) and striping counts."""
import pytest

pytestmark = pytest.mark.gpu

KEYS = ("dep_L", "dep_U", "dep_U_row", "dep_U_rowcol", "cond_L", "cond_U", "striping_flagged", "nnz_L", "nnz_U")


@pytest.mark.parametrize("spec", ["poisson2d(24,24)", "poisson3d(12,12,12)", "cutcell(16,16,16)",
                                  "pressure27(12,12,12)"])
@pytest.mark.parametrize("kv", [{}, {"ilu.variant": "ilut"}, {"scaling": "none"}, {"scaling": "row_col"}],
                         ids=["ilu0-row", "ilut-row", "ilu0-none", "ilu0-rowcol"])
def test_run_analyze_matches_reference(ilug, ref, torch_cuda, spec, kv):
    A = ilug.Matrix.generate(spec)
    rep = ilug.run_analyze(A, ilug.Config().update(kv))
    want = ref.run_analyze(A.csr(), kv)
    for k in KEYS:
        assert rep[k] == want[k], (k, rep[k], want[k])
    assert "analyze" in rep.tables


def test_c3_departure_collapse(ilug, torch_cuda):
    """Table-1 effect on the cut-cell matrix: row scaling collapses dep(U) by many
    orders of magnitude (dep(D^-1 U) is O(10^2) while dep(U) is O(10^16))."""
    rep = ilug.run_analyze(ilug.Matrix.generate("cutcell(32,32,32)"), ilug.Config())
    assert float(rep["dep_U"]) > 1e12 * float(rep["dep_U_row"])
