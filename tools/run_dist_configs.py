"""Iteration counts of the row-block distributed solve vs the rank count at
the BASELINE sizes (not a test, not the bench): p ranks as host threads on
the one GPU through the in-process transport (the NCCL path's kernels and
plans; wall times here are NOT multi-GPU timings — every collective
synchronises and the ranks share one GPU).

    python tools/run_dist_configs.py [c4] [c5] [P ...]

c4: poisson3d(465^3) (100.5 M rows), block-Jacobi ILU(0) m = 5,5, poly-GS below,
    GMRES relres 1e-8 — BASELINE configs[3]
c5: pressure27(64^3) and poisson3d(64^3), ILUT Schur-complement smoother with
    schur.blocks = p, FGMRES — BASELINE configs[4]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_09512_b200 as ilug  # noqa: E402
from paper_2111_09512_b200 import dist as idist  # noqa: E402

args = sys.argv[1:]
which = [a for a in args if a.startswith("c")] or ["c4", "c5"]
ps = [int(a) for a in args if a.isdigit()] or [1, 2, 4, 8]


def run(spec, kv, p, label):
    A = ilug.Matrix.generate(spec)
    cfg = ilug.Config().update(kv)
    t = time.time()
    H = ilug.Hierarchy(A, ilug.Config().update(dict(kv, **{"device.amg_setup": "device"})), host_only=True)
    host_s = time.time() - t
    rp, _, v = A.csr()
    group = idist.LocalGroup(p)

    def rank(r):
        comm = group.comm(r)
        t0 = time.time()
        S = idist.Solver(H, comm)
        setup = time.time() - t0
        r0, r1 = S.row0, S.row0 + S.nloc
        b = torch.from_numpy(np.add.reduceat(v[:rp[r1]], rp[r0:r1])).cuda()  # b = A * ones
        x = torch.zeros_like(b)
        torch.cuda.synchronize()
        t0 = time.time()
        out = S.gmres(cfg, b, x)
        torch.cuda.synchronize()
        return dict(out, setup_s=setup, solve_s=time.time() - t0, levels=S.levels)

    res = idist.run_ranks(p, rank, group)
    its = {o["iterations"] for o in res}
    print(json.dumps({"config": label, "spec": spec, "ranks": p, "iterations": its.pop() if len(its) == 1 else sorted(its),
                      "converged": all(o["status"] == 0 for o in res), "final_relres": res[0]["final_relres"],
                      "levels": res[0]["levels"], "host_hierarchy_s": round(host_s, 2),
                      "rank_setup_s_max": round(max(o["setup_s"] for o in res), 2),
                      "solve_s_one_gpu_inprocess": round(max(o["solve_s"] for o in res), 2)}), flush=True)


if "c4" in which:
    kv = {"smoother.kind": "ilu", "ilu.variant": "ilu0", "scaling": "row", "trisolve.m_lower": "5",
          "trisolve.m_upper": "5", "smoother.sweeps": "2", "smoother.fallback.kind": "poly_gs",
          "amg.coarsening": "pmis", "krylov.tol": "1e-8", "krylov.form_iterates": "false"}
    for p in ps:
        run("poisson3d(465,465,465)", kv, p, "C4 block-Jacobi ILU(0) GMRES+AMG")
if "c5" in which:
    for spec in ("poisson3d(64,64,64)", "pressure27(64,64,64)"):
        for p in ps:
            kv = {"smoother.kind": "schur_ilut", "schur.blocks": str(p), "krylov.method": "fgmres",
                  "amg.coarsening": "pmis", "krylov.tol": "1e-8", "krylov.form_iterates": "false"}
            run(spec, kv, p, "C5 Schur-complement smoother FGMRES+AMG")
