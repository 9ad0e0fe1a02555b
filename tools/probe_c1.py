import os, sys, time
sys.path.insert(0, '/root/repo') if os.path.exists('/root/repo') else None
sys.path.insert(0, os.getcwd())
import paper_2111_09512_b200 as ilug
kv = {"smoother.kind": "ilu", "ilu.variant": "ilu0", "scaling": "row", "trisolve.mode": "richardson",
      "trisolve.m_lower": "5", "trisolve.m_upper": "5", "smoother.sweeps": "2",
      "smoother.fallback.kind": "gauss_seidel", "amg.coarsening": "pmis", "krylov.tol": "1e-8"}
A = ilug.Matrix.generate("poisson3d(64,64,64)")
for extra in ({}, {"krylov.form_iterates": "false"}, {"smoother.fallback.kind": "poly_gs"},
              {"smoother.fallback.kind": "poly_gs", "krylov.form_iterates": "false"}):
    cfg = ilug.Config().update(dict(kv, **extra))
    ilug.run_solve(A, cfg)
    rep = ilug.run_solve(A, cfg)
    print(extra, rep["iterations"], rep["setup_seconds"], rep["solve_seconds"], rep["device_vcycles"], flush=True)
H = ilug.Hierarchy(A, ilug.Config().update(kv))
print("levels", H.levels, [H.level_matrix(k).rows for k in range(H.levels)], flush=True)
import torch
r = torch.rand(A.rows, dtype=torch.float64, device="cuda"); z = torch.empty_like(r)
for _ in range(3): H.vcycle(r, z)
torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): H.vcycle(r, z)
e1.record(); torch.cuda.synchronize(); print("vcycle ms", e0.elapsed_time(e1) / 20, "graph nodes", H.graph_nodes, flush=True)
os.environ["ILUG_TRACE"] = "1"
H2 = ilug.Hierarchy(A, ilug.Config().update(dict(kv, **{"device.graph": "false"})))
H2.vcycle(r, z); torch.cuda.synchronize()
