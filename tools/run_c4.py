"""C4-size single-GPU data point (not the bench): GMRES+AMG on the 465^3
7-point Poisson matrix (100.5 M rows) through iluamg_run_solve, iterative vs
level-scheduled direct triangular solves; prints one JSON line per mode.

    python tools/run_c4.py [SPEC] [modes]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "poisson3d(465,465,465)"
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["richardson", "direct"]
kv = {"smoother.kind": "ilu", "ilu.variant": "ilu0", "trisolve.m_lower": "5", "trisolve.m_upper": "5",
      "smoother.sweeps": "2", "krylov.tol": "1e-8", "amg.coarsening": "pmis", "krylov.form_iterates": "false",
      "smoother.fallback.kind": "poly_gs"}
t = time.time()
A = ilug.Matrix.generate(spec)
gen = time.time() - t
for mode in modes:
    ilug.run_solve(ilug.Matrix.generate("poisson3d(24,24,24)"), ilug.Config().update(dict(kv, **{"trisolve.mode": mode})))
    t = time.time()
    rep = ilug.run_solve(A, ilug.Config().update(dict(kv, **{"trisolve.mode": mode})))
    print(json.dumps({"spec": spec, "n": A.rows, "nnz": A.nnz, "mode": mode, "generate_s": round(gen, 1),
                      "wall_s": round(time.time() - t, 1), "iterations": int(rep["iterations"]),
                      "converged": rep["converged"], "setup_s": float(rep["setup_seconds"]),
                      "solve_s": float(rep["solve_seconds"]), "final_relres": float(rep["final_relres"]),
                      "levels": int(rep["levels"]), "vcycles": int(rep["device_vcycles"])}), flush=True)
