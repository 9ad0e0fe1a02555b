"""Time of the coarse part of the C2 V-cycle (levels >= 1) in graph replay:
a hierarchy built on the level-1 operator with the same coarse smoother (not
a test)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_09512_b200 as ilug  # noqa: E402

kv = {"smoother.kind": "poly_gs", "smoother.sweeps": "2", "amg.coarsening": "pmis",
      "smoother.fallback.kind": "poly_gs"}
A = ilug.Matrix.generate(sys.argv[1] if len(sys.argv) > 1 else "pressure27(256,256,256)")
H0 = ilug.Hierarchy(A, ilug.Config().update({"amg.coarsening": "pmis"}), host_only=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for lvl in range(1, min(4, H0.levels)):
    A1 = H0.level_matrix(lvl, "A")
    for graph in (True, False):
        H = ilug.Hierarchy(A1, ilug.Config().update(dict(kv, **{"device.graph": graph})))
        r = torch.rand(A1.rows, dtype=torch.float64, device="cuda")
        z = torch.empty_like(r)
        for _ in range(3):
            H.vcycle(r, z)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            H.vcycle(r, z)
        e1.record()
        torch.cuda.synchronize()
        print(f"from level {lvl} (n={A1.rows}, {H.levels} levels) graph={graph}: {e0.elapsed_time(e1) / 20:.3f} ms "
              f"nodes={H.graph_nodes}", flush=True)
