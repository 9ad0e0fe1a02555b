"""Data points for the BASELINE.json configs other than the bench's C2 line
(not a test, not the bench); one JSON object per config on stdout.

    python tools/run_configs.py [c1] [c3] [c5]

c1: 7-point 64^3 ILU(0): unscaled vs row-scaled U, 5 sweeps vs the direct
    solve (error to direct, device time per sweep; the reference's own CPU
    figures are in SURVEY.md §8a).
c3: cut-cell 256^3 (coefficient jumps over 16 decades): dep(U) vs dep(D^-1 U)
    at 64^3 via run_analyze, and at 256^3 scaled vs unscaled-Jacobi sweep time
    and error to the direct solve for m = 5, 20, 40.
c5: ILUT Schur-complement smoother under FGMRES (run_schur_solve) on
    pressure27(64^3): iterations and time for 1, 2, 4, 8 sub-domains."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_09512_b200 as ilug  # noqa: E402

which = sys.argv[1:] or ["c1", "c3", "c5"]
torch.cuda.set_device(0)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps


def rel(a, b):
    return float(torch.linalg.norm(a - b) / torch.linalg.norm(b))


def sweeps(spec, ms):
    A = ilug.Matrix.generate(spec)
    t = time.time()
    L, U = ilug.ilu_factorize_device(A, ilug.Config())
    tf = time.time() - t
    Lc, Uc = L.csr(), U.csr()
    fs = ilug.Factors.from_csr(A.rows, Lc, Uc, scaling="row", direct=True)
    fj = ilug.Factors.from_csr(A.rows, Lc, Uc, scaling="row", upper="jacobi")
    b = torch.rand(A.rows, dtype=torch.float64, device="cuda") * 2 - 1
    xd, xs, xj = (torch.empty_like(b) for _ in range(3))
    fs.solve_upper(b, xd)
    out = {"spec": spec, "n": A.rows, "nnz_U": int(U.nnz), "factor_s": round(tf, 2),
           "direct_upper_ms": round(timed(lambda: fs.solve_upper(b, xd), 5), 3), "m": {}}
    for m in ms:
        ts = timed(lambda: fs.sweep_upper(b, xs, m))
        tj = timed(lambda: fj.sweep_upper(b, xj, m))
        out["m"][m] = {"scaled_ms": round(ts, 3), "jacobi_ms": round(tj, 3),
                       "scaled_err_vs_direct": rel(xs, xd), "jacobi_vs_scaled": rel(xj, xs)}
    return out


if "c1" in which:
    print(json.dumps({"config": "C1 poisson3d(64,64,64) ILU(0)", **sweeps("poisson3d(64,64,64)", [5, 10])}),
          flush=True)
if "c3" in which:
    an = ilug.run_analyze(ilug.Matrix.generate("cutcell(64,64,64)"), ilug.Config())
    keys = ("dep_L", "dep_U", "dep_U_row", "dep_U_rowcol")
    print(json.dumps({"config": "C3 cutcell(64^3) departures (run_analyze)",
                      **{k: an.scalars[k] for k in keys if k in an.scalars}}), flush=True)
    print(json.dumps({"config": "C3 cutcell(256,256,256) ILU(0)", **sweeps("cutcell(256,256,256)", [5, 20, 40])}),
          flush=True)
if "c5" in which:
    spec = "pressure27(64,64,64)"
    A = ilug.Matrix.generate(spec)
    t = time.time()
    rep = ilug.run_schur_solve(A, ilug.Config().update({"krylov.tol": "1e-8"}))
    res = {"config": "C5 schur_ilut FGMRES " + spec, "n": A.rows, "wall_s": round(time.time() - t, 1),
           "scalars": dict(rep.scalars), "tables": dict(rep.tables)}
    print(json.dumps(res), flush=True)
