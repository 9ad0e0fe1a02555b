"""One Gauss-Seidel sweep on one coarse level of SPEC's PMIS hierarchy (an ncu
target for the level-scheduled K5 kernels; not a test).

    python tools/probe_gs_level.py [SPEC] [LEVEL]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "pressure27(256,256,256)"
lvl = int(sys.argv[2]) if len(sys.argv) > 2 else 2
A = ilug.Matrix.generate(spec)
H = ilug.Hierarchy(A, ilug.Config().update({"amg.coarsening": "pmis"}), host_only=True)
M = H.level_matrix(lvl, "A")
S = ilug.Smoother(M, ilug.Config().update({"smoother.kind": "gauss_seidel", "smoother.sweeps": "1"}))
b = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, M.rows)).cuda()
x = torch.zeros_like(b)
S.smooth(b, x)
torch.cuda.synchronize()
print("level", lvl, "rows", M.rows, flush=True)
