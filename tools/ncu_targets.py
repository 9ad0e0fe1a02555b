"""Single launches of the hot kernels on the C2 ILUT(1e-3,5) factors, for ncu
(`-k regex:... -c 1`); not a test, not the bench.

    python tools/ncu_targets.py u|l|k5u|k5l [SPEC]

u / l: one scaled-U / L Richardson sweep kernel (k_rowdot<EpiResidual>, the
bench's dominant kernel); k5u / k5l: one level-scheduled direct solve (K5)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_09512_b200 as ilug  # noqa: E402

what = sys.argv[1]  # u | l | k5u | k5l | step (one ilu_smooth_sweep: residual, L sweeps, U sweeps, x += ...)
spec = sys.argv[2] if len(sys.argv) > 2 else "pressure27(256,256,256)"
kv = {"ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5"}
torch.cuda.set_device(0)
A = ilug.Matrix.generate(spec)
if what == "step":
    S = ilug.Smoother(A, ilug.Config().update(dict(kv, **{"smoother.kind": "ilu", "trisolve.m_lower": "5",
                                                          "trisolve.m_upper": "5"})))
else:
    F = ilug.Factors.create(A, ilug.Config().update(kv), scaling="row", direct=what.startswith("k5"))
n = A.rows
b = torch.rand(n, dtype=torch.float64, device="cuda")
out = torch.empty_like(b)
torch.cuda.synchronize()
if what == "u":
    F.sweep_upper(b, out, 3)  # scale, one residual sweep (k_rowdot<EpiResidual>), the accumulate sweep
elif what == "l":
    F.sweep_lower(b, out, 3)
elif what == "k5u":
    F.solve_upper(b, out)
elif what == "k5l":
    F.solve_lower(b, out)
elif what == "step":
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    for _ in range(int(os.environ.get("NCU_REPS", "1"))):  # NCU_REPS > 1: warm repeats (take the last)
        S.ilu_sweep(b, x)
torch.cuda.synchronize()
print("done", what)
