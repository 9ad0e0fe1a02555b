import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2111_09512_b200 as ilug
from oracle import oracle
r = oracle.Ref()
spec, p = sys.argv[1], sys.argv[2]
kv = {"smoother.kind": "schur_ilut", "schur.blocks": p, "krylov.method": "fgmres"}
A = ilug.Matrix.generate(spec)
rng = np.random.default_rng(7)
rv = rng.uniform(-1, 1, A.rows)
Ar = r.mat(*A.csr())
H = r.amg(Ar, r.cfg(kv))
want = r.vcycle(H, rv, np.zeros(A.rows))
print("ref vcycle finite", np.isfinite(want).all(), "levels", r.amg_levels(H), flush=True)
for graph in (True, False):
    Hd = ilug.Hierarchy(A, ilug.Config().update(kv).set("device.graph", graph))
    for rep in range(3):
        z = torch.empty(A.rows, dtype=torch.float64, device="cuda")
        Hd.vcycle(torch.from_numpy(rv).cuda(), z)
        got = z.cpu().numpy()
        d = np.abs(got - want)
        print("graph", graph, "rep", rep, "finite", np.isfinite(got).all(), "max rel diff",
              float(np.nanmax(d) / np.abs(want).max()), "levels", Hd.levels, flush=True)
