import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2111_09512_b200 as ilug
spec, p = sys.argv[1], sys.argv[2]
A = ilug.Matrix.generate(spec)
rng = np.random.default_rng(7)
bv = rng.uniform(-1, 1, A.rows)
for method in ("fgmres", "gmres"):
    for graph in (True, False):
        for fi in ("true", "false"):
            kv = {"smoother.kind": "schur_ilut", "schur.blocks": p, "krylov.method": method, "krylov.tol": "1e-8",
                  "device.graph": graph, "krylov.form_iterates": fi, "krylov.max_iters": "60"}
            H = ilug.Hierarchy(A, ilug.Config().update(kv))
            x = torch.zeros(A.rows, dtype=torch.float64, device="cuda")
            try:
                out = H.gmres(ilug.Config().update(kv), torch.from_numpy(bv).cuda(), x)
                print(method, "graph", graph, "form_iterates", fi, out, flush=True)
            except ilug.IlugError as e:
                print(method, "graph", graph, "form_iterates", fi, "ERR", e, flush=True)
