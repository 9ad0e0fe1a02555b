"""Debug probe: V-cycle parity on poisson2d(40,40) for both level-set schedules."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_09512_b200 as ilug  # noqa: E402
from oracle import oracle  # noqa: E402

ref = oracle.Ref()
spec = sys.argv[1] if len(sys.argv) > 1 else "poisson2d(40,40)"
kv = {"smoother.kind": "ilu", "trisolve.m_lower": 5, "trisolve.m_upper": 5}
A = ilug.Matrix.generate(spec)
Ar = ref.mat(*A.csr())
Hr = ref.amg(Ar, ref.cfg(kv))
r = np.random.default_rng(1).uniform(-1, 1, A.rows)
want = ref.vcycle(Hr, r, np.zeros(A.rows))
for sched in ("cta", "flags"):
    os.environ["ILUG_LEVELSET"] = sched
    H = ilug.Hierarchy(A, ilug.Config().update(kv).set("device.graph", False))
    z = torch.empty(A.rows, dtype=torch.float64, device="cuda")
    H.vcycle(torch.from_numpy(r).cuda(), z)
    torch.cuda.synchronize()
    got = z.cpu().numpy()
    print(sched, "levels", H.levels, "bitwise", np.array_equal(got, want), "maxdiff", np.abs(got - want).max())
    for k in range(H.levels):
        M = H.level_matrix(k, "A")
        print("  level", k, M.rows, M.nnz)
    # GS sweep alone on each level matrix
    for k in range(1, H.levels - 1):
        Mk = H.level_matrix(k, "A")
        S = ilug.Smoother(Mk, ilug.Config().set("smoother.kind", "gauss_seidel"))
        Mr = ref.mat(*Mk.csr())
        Sr = ref.smoother(Mr, ref.cfg({"smoother.kind": "gauss_seidel"}))
        b = np.random.default_rng(k).uniform(-1, 1, Mk.rows)
        x0 = np.random.default_rng(k + 9).uniform(-1, 1, Mk.rows)
        xd = torch.from_numpy(x0).cuda()
        S.smooth(torch.from_numpy(b).cuda(), xd)
        torch.cuda.synchronize()
        w, _ = ref.smooth(Mr, Sr, b, x0)
        print("   GS level", k, "bitwise", np.array_equal(xd.cpu().numpy(), w), np.abs(xd.cpu().numpy() - w).max())
