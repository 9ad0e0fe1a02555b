"""Diagnostics for the GMRES+AMG solve on the device (not a test, not the bench).

    python tools/probe_tts.py SPEC [key=value ...]

Prints the hierarchy, the V-cycle time (graph replay), one eager V-cycle with
ILUG_TRACE per-level phase times, the direct-solve residual check of the
finest ILU factors, and one GMRES solve."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "pressure27(128,128,128)"
kv = {"smoother.kind": "ilu", "ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5",
      "trisolve.m_lower": "5", "trisolve.m_upper": "5", "krylov.tol": "1e-8", "amg.coarsening": "pmis",
      "krylov.form_iterates": "false"}
for a in sys.argv[2:]:
    k, v = a.split("=", 1)
    kv[k] = v
torch.cuda.set_device(0)
t = time.time()
A = ilug.Matrix.generate(spec)
print(f"generate {time.time() - t:.2f}s n={A.rows} nnz={A.nnz}", flush=True)
cfg = ilug.Config().update(kv)
t = time.time()
H = ilug.Hierarchy(A, cfg)
print(f"hierarchy setup {time.time() - t:.2f}s levels={H.levels} oc={H.operator_complexity:.3f}", flush=True)
for k in range(H.levels):
    M = H.level_matrix(k, "A")
    print(f"  level {k}: n={M.rows} nnz={M.nnz} ({M.nnz / max(M.rows, 1):.1f}/row)")
n = A.rows
r = torch.rand(n, dtype=torch.float64, device="cuda")
z = torch.empty_like(r)
H.vcycle(r, z)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    H.vcycle(r, z)
e1.record()
torch.cuda.synchronize()
print(f"vcycle (graph) {e0.elapsed_time(e1) / 5:.3f} ms, graph nodes {H.graph_nodes}", flush=True)
os.environ["ILUG_TRACE"] = "1"
He = ilug.Hierarchy(A, ilug.Config().update(kv).set("device.graph", False))
He.vcycle(r, z)
torch.cuda.synchronize()
del He
# direct-solve residual check of the finest factors
F = ilug.Factors.create(A, cfg, scaling="row", direct=True)
print("factor stats", F.stats(), flush=True)
b = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
x = torch.empty_like(b)
F.solve_upper(b, x)
torch.cuda.synchronize()
(rp, ci, v), rs, _ = F.download_upper()
U = ilug.Matrix.from_csr(n, n, rp, ci, v)
DU = ilug.DeviceMatrix(U)
y = torch.empty_like(b)
DU.spmv(x, y)
bs = b.cpu().numpy() / rs
print("upper direct residual rel", float(np.linalg.norm(y.cpu().numpy() - bs) / np.linalg.norm(bs)),
      "|x|/|bs|", float(x.norm()) / float(np.linalg.norm(bs)), flush=True)
for m in (5, 10, 20):
    F.sweep_upper(b, y, m)
    torch.cuda.synchronize()
    print(f"  richardson m={m} rel diff to direct", float((y - x).norm() / x.norm()), flush=True)
t = time.time()
rep = ilug.run_solve(A, cfg)
print(f"run_solve {time.time() - t:.1f}s iterations={rep['iterations']} setup={rep['setup_seconds']} "
      f"solve={rep['solve_seconds']} relres={rep['final_relres']} vcycles={rep['device_vcycles']}", flush=True)
