import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2111_09512_b200 as ilug
from oracle import oracle
r = oracle.Ref()
SCHUR = {"smoother.kind": "schur_ilut", "smoother.sweeps": "1"}
spec = sys.argv[1]
A = ilug.Matrix.generate(spec)
Ar = r.mat(*A.csr())
rng = np.random.default_rng(5)
b, x0 = rng.uniform(-1, 1, A.rows), rng.uniform(-1, 1, A.rows)
for p in sys.argv[2].split(","):
    kv = dict(SCHUR, **{"schur.blocks": p})
    want, _ = r.smooth(Ar, r.smoother(Ar, r.cfg(kv)), b, x0)
    S = ilug.Smoother(A, ilug.Config().update(kv))
    for rep in range(3):
        xd = torch.from_numpy(x0.copy()).cuda()
        S.smooth(torch.from_numpy(b).cuda(), xd)
        got = xd.cpu().numpy()
        d = np.abs(got - want)
        print(spec, "p", p, "rep", rep, "finite", np.isfinite(got).all(), "max rel diff", float(np.nanmax(d) / np.abs(want).max()),
              "n differ", int((d > 0).sum()), flush=True)
