"""One C2 V-cycle (eager launches) for a per-kernel launch list under ncu
(not a test): python tools/probe_vcycle.py [SPEC]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "pressure27(256,256,256)"
kv = {"smoother.kind": "ilu", "ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5",
      "trisolve.m_lower": "5", "trisolve.m_upper": "5", "smoother.sweeps": "2", "amg.coarsening": "pmis",
      "smoother.fallback.kind": "poly_gs", "device.graph": "false"}
A = ilug.Matrix.generate(spec)
H = ilug.Hierarchy(A, ilug.Config().update(kv))
r = torch.rand(A.rows, dtype=torch.float64, device="cuda")
z = torch.empty_like(r)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
H.vcycle(r, z)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("levels", H.levels)
