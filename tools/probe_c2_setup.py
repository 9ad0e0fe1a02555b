"""C2 GMRES+AMG solve through run_solve with ILUG_TRACE_SETUP phase times on
stderr (setup breakdown: host AMG levels, device factorisation); not a test.

    python tools/probe_c2_setup.py [SPEC] [key=value ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if "ILUG_TRACE_SETUP" not in os.environ:
    os.environ["ILUG_TRACE_SETUP"] = "1"
import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "pressure27(256,256,256)"
kv = {"smoother.kind": "ilu", "ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5",
      "trisolve.m_lower": "5", "trisolve.m_upper": "5", "krylov.tol": "1e-8", "amg.coarsening": "pmis",
      "smoother.fallback.kind": "poly_gs", "smoother.sweeps": "2",
      "krylov.form_iterates": "false"}
kv.update(dict(a.split("=", 1) for a in sys.argv[2:]))
t = time.time()
A = ilug.Matrix.generate(spec)
print(f"generate {time.time() - t:.2f}s n={A.rows} nnz={A.nnz} cores={os.cpu_count()}", file=sys.stderr, flush=True)
ilug.run_solve(ilug.Matrix.generate("pressure27(16,16,16)"), ilug.Config().update(kv))  # warm-up
t = time.time()
rep = ilug.run_solve(A, ilug.Config().update(kv))
print(f"run_solve wall {time.time() - t:.2f}s setup {rep['setup_seconds']} solve {rep['solve_seconds']} "
      f"iterations {rep['iterations']}", file=sys.stderr, flush=True)
