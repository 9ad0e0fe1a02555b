"""Reference GMRES+AMG results at the BASELINE configurations, computed by the
REFERENCE ITSELF (oracle/_ref run_solve = src/driver.cpp:239-260) in the build
container and committed as tests/golden/baseline_solves.json.

    python tests/golden/make_baseline_solves.py [-j JOBS]

The reference is single-threaded and needs minutes for the C2-family slab, so
the GPU tests (tests/test_gpu_baseline.py) compare the device's counts with
these fixtures instead of re-running the reference on the box. Each record
holds the spec, the exact config keys, the reference's iterations / status /
final relres / levels and a SHA-256 of the generated CSR (a generator change
is caught before a count is compared).

Configs (BASELINE.json `configs`):
  C1  poisson3d(64^3)  ilu0, m_L=m_U=5, sweeps 2, GS fallback, PMIS, tol 1e-8;
      row-scaled Richardson (reference: 13 its), row_col Richardson, direct
      (row) and direct on unscaled factors.
  C3  cutcell(64^3)    the same four factor/scaling variants.
  C2s pressure27(256,256,16) (a 16-plane slab of C2): ILUT(1e-3,5), PMIS,
      Richardson m=5,5 with the GS and the poly-GS coarse fallback, and direct.
"""
import argparse
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

BASE = {"smoother.kind": "ilu", "ilu.variant": "ilu0", "trisolve.m_lower": "5", "trisolve.m_upper": "5",
        "smoother.sweeps": "2", "smoother.fallback.kind": "gauss_seidel", "amg.coarsening": "pmis",
        "krylov.tol": "1e-8"}
VARIANTS = {
    "row_richardson": {"scaling": "row", "trisolve.mode": "richardson"},
    "rowcol_richardson": {"scaling": "row_col", "trisolve.mode": "richardson"},
    "row_direct": {"scaling": "row", "trisolve.mode": "direct"},
    "none_direct": {"scaling": "none", "trisolve.mode": "direct"},
}
ILUT = {"ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5"}

CASES = {}
for spec, tag in (("poisson3d(64,64,64)", "C1"), ("cutcell(64,64,64)", "C3")):
    for v, kv in VARIANTS.items():
        CASES[f"{tag}|{v}"] = (spec, dict(BASE, **kv))
SLAB = "pressure27(256,256,16)"
CASES["C2s|row_richardson|gs"] = (SLAB, dict(BASE, **ILUT, **VARIANTS["row_richardson"]))
CASES["C2s|row_richardson|poly_gs"] = (SLAB, dict(BASE, **ILUT, **VARIANTS["row_richardson"],
                                                  **{"smoother.fallback.kind": "poly_gs"}))
CASES["C2s|row_direct|gs"] = (SLAB, dict(BASE, **ILUT, **VARIANTS["row_direct"]))


def csr_sha(csr):
    return hashlib.sha256(b"".join(a.tobytes() for a in csr)).hexdigest()


def run(key):
    import paper_2111_09512_b200 as ilug  # host generator only (the matrix both sides see)
    from oracle import oracle
    spec, kv = CASES[key]
    csr = ilug.Matrix.generate(spec).csr()
    t = time.time()
    out = oracle.Ref().run_solve(csr, kv)
    return key, {"spec": spec, "kv": kv, "A_sha": csr_sha(csr), "iterations": int(out["iterations"]),
                 "converged": out["converged"], "status": out["status"],
                 "final_relres": float(out["final_relres"]), "levels": int(out["levels"]),
                 "setup_seconds": float(out["setup_seconds"]), "solve_seconds": float(out["solve_seconds"]),
                 "wall_s": round(time.time() - t, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=os.cpu_count())
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    path = os.path.join(HERE, "baseline_solves.json")
    res = json.load(open(path)) if os.path.exists(path) else {}
    keys = [k for k in CASES if not a.only or a.only in k]
    with ProcessPoolExecutor(a.j) as ex:
        for key, rec in ex.map(run, keys):
            res[key] = rec
            print(key, rec["iterations"], rec["converged"], rec["wall_s"], flush=True)
            with open(path, "w") as fh:
                json.dump(res, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
