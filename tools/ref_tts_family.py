"""Time-to-solution next to the reference's CPU path at a size the reference
finishes ("time ... the full solve at 128^3/256^3, and state the
extrapolation"): the C4 configuration (7-point Poisson, ILU(0) row-scaled,
m = 5,5, 2 sweeps, PMIS, poly-GS fallback, relres 1e-8) and the C2
configuration (pressure27, ILUT(1e-3,5)) through iluamg_run_solve on the GPU
and through the reference's run_solve on one host core (the reference is
single-threaded), on the same matrix (oracle-side generator for the
reference). Not a test; prints one JSON line per case.

    python tools/ref_tts_family.py [N ...]   (grid edge, default 128)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_09512_b200 as ilug  # noqa: E402
from oracle import oracle  # noqa: E402

BASE = {"smoother.kind": "ilu", "scaling": "row", "trisolve.mode": "richardson", "trisolve.m_lower": "5",
        "trisolve.m_upper": "5", "smoother.sweeps": "2", "smoother.fallback.kind": "poly_gs",
        "amg.coarsening": "pmis", "krylov.tol": "1e-8"}
CASES = {"C4-family": ("poisson3d({0},{0},{0})", {"ilu.variant": "ilu0"}),
         "C2-family": ("pressure27({0},{0},{0})", {"ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5"})}
ref = oracle.Ref()
for edge in [int(a) for a in sys.argv[1:]] or [128]:
    for name, (fmt, extra) in CASES.items():
        spec = fmt.format(edge)
        kv = dict(BASE, **extra)
        A = ilug.Matrix.generate(spec)
        ilug.run_solve(ilug.Matrix.generate(fmt.format(16)), ilug.Config().update(kv))  # warm-up
        d = ilug.run_solve(A, ilug.Config().update(kv))
        t = time.time()
        r = ref.run_solve(ref.arrays(ref.gen3d(spec)), kv)
        wall = time.time() - t
        print(json.dumps({"case": name, "spec": spec, "device": {"iterations": int(d["iterations"]),
                          "setup_s": float(d["setup_seconds"]), "solve_s": float(d["solve_seconds"])},
                          "reference_1core": {"iterations": int(r["iterations"]), "setup_s": float(r["setup_seconds"]),
                                              "solve_s": float(r["solve_seconds"]), "wall_s": round(wall, 1)},
                          "speedup_solve": round(float(r["solve_seconds"]) / float(d["solve_seconds"]), 1),
                          "speedup_total": round((float(r["setup_seconds"]) + float(r["solve_seconds"])) /
                                                 (float(d["setup_seconds"]) + float(d["solve_seconds"])), 1)}),
              flush=True)
