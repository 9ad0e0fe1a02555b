import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2111_09512_b200 as ilug
from oracle import oracle
r = oracle.Ref()
for spec in sys.argv[1:]:
    A = ilug.Matrix.generate(spec)
    Ar = r.mat(*A.csr())
    rng = np.random.default_rng(5)
    b, x0 = rng.uniform(-1, 1, A.rows), rng.uniform(-1, 1, A.rows)
    want, _ = r.smooth(Ar, r.smoother(Ar, r.cfg({"smoother.kind": "gauss_seidel"})), b, x0)
    for sched in ("cta", "flags", None):
        if sched: os.environ["ILUG_LEVELSET"] = sched
        else: os.environ.pop("ILUG_LEVELSET", None)
        S = ilug.Smoother(A, ilug.Config().set("smoother.kind", "gauss_seidel"))
        bad = 0
        for rep in range(5):
            xd = torch.from_numpy(x0.copy()).cuda()
            S.smooth(torch.from_numpy(b).cuda(), xd)
            got = xd.cpu().numpy()
            if not np.array_equal(got.view(np.int64), want.view(np.int64)):
                bad += 1
                d = np.abs(got - want); print("  mismatch rep", rep, "max diff", d.max(), "n bad", (d > 0).sum(), "first", np.argmax(d > 0))
        print(spec, "sched", sched, "mismatches", bad, "of 5", flush=True)
