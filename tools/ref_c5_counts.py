"""Reference iteration counts for the C5 configuration (Schur-complement ILUT
smoother with p blocks under FGMRES+AMG, b = A*1) from the composed
reference (oracle/_ref: the reference's own Schur smoother with p blocks and
block smoothers below), on the CPU of this container. Not a test; prints one
JSON line per (spec, p) to compare with profiles/r02_dist_configs.jsonl.

    python tools/ref_c5_counts.py SPEC p1 [p2 ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as _o  # noqa: E402

ref = _o.Ref()
spec = sys.argv[1]
A = ref.gen3d(spec)
rp, ci, v = ref.arrays(A)
b = np.add.reduceat(v, rp[:-1]) if len(v) else np.zeros(len(rp) - 1)
for p in map(int, sys.argv[2:]):
    kv = {"smoother.kind": "schur_ilut", "schur.blocks": str(p), "krylov.method": "fgmres",
          "amg.coarsening": "pmis", "krylov.tol": "1e-8"}
    t = time.time()
    d = ref.dist_setup(A, ref.cfg(kv), p)
    out = ref.dist_krylov(A, d, ref.cfg(kv), b)
    print(json.dumps({"spec": spec, "ranks": p, "reference_iterations": out["iterations"],
                      "converged": out["converged"], "seconds": round(time.time() - t, 1)}), flush=True)
