"""One Gauss-Seidel sweep (K5 level-set kernel) on a coarse AMG operator of
SPEC's hierarchy, timed with CUDA events, for ncu targeting; not a test.

    python tools/probe_gs.py [SPEC] [LEVEL]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "pressure27(128,128,128)"
lvl = int(sys.argv[2]) if len(sys.argv) > 2 else 2
A = ilug.Matrix.generate(spec)
H = ilug.Hierarchy(A, ilug.Config().update({"amg.coarsening": "pmis"}), host_only=True)
M = H.level_matrix(lvl, "A")
S = ilug.Smoother(M, ilug.Config().update({"smoother.kind": "gauss_seidel", "smoother.sweeps": "1"}))
b = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, M.rows)).cuda()
x = torch.zeros_like(b)
for _ in range(3):
    S.smooth(b, x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    S.smooth(b, x)
e1.record()
torch.cuda.synchronize()
print(f"level {lvl}: n={M.rows} nnz={M.nnz} GS sweep {e0.elapsed_time(e1) / 10:.3f} ms", flush=True)
