"""Same-process A/B of eager C2 V-cycles under an env knob (not a test):
    PROBE_VAR=ILUG_ROWDOT_HOIST PROBE_VALS=0,1,0,1 python tools/probe_vcycle_ab.py [SPEC]
The knobs are read per launch, so graph capture is off (device.graph=false)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "pressure27(256,256,256)"
kv = {"smoother.kind": "ilu", "ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5",
      "trisolve.m_lower": "5", "trisolve.m_upper": "5", "smoother.sweeps": "2", "amg.coarsening": "pmis",
      "smoother.fallback.kind": os.environ.get("PROBE_FALLBACK", "poly_gs"), "device.graph": "false"}
A = ilug.Matrix.generate(spec)
H = ilug.Hierarchy(A, ilug.Config().update(kv))
r = torch.rand(A.rows, dtype=torch.float64, device="cuda")
z = torch.empty_like(r)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
var = os.environ.get("PROBE_VAR", "ILUG_ROWDOT_HOIST")
ref = None
for v in os.environ.get("PROBE_VALS", "0,1,0,1,0,1").split(","):
    os.environ[var] = v
    for _ in range(3):
        H.vcycle(r, z)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        H.vcycle(r, z)
    e1.record()
    torch.cuda.synchronize()
    same = ref is None or torch.equal(ref, z)
    ref = z.clone() if ref is None else ref
    print(f"{var}={v} levels={H.levels} vcycle {e0.elapsed_time(e1) / 20:.3f} ms bitwise_same={same}", flush=True)
