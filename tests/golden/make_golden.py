"""Regenerate the golden fixtures from the REFERENCE ITSELF (oracle/_ref).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Each fixture holds a seeded input and the reference library's outputs for the
hot path (row_scale + richardson_upper_scaled, richardson_lower,
solve_upper_scaled_direct) on one generated matrix, plus a hash of the matrix
so a generator change is caught. The GPU tests and the port tests compare
against these bitwise, so parity stays pinned even where oracle/_ref is absent.
Also writes solve_counts.json: the reference's GMRES+AMG iteration counts for
the solve configurations of tests/test_gpu_solver.py.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import paper_2111_09512_b200 as ilug  # noqa: E402  (host setup only: generator)
from oracle import oracle  # noqa: E402

CASES = [
    ("c1_poisson3d_16", "poisson3d(16,16,16)", {}, 5, 101),
    ("c2_pressure27_10_ilut", "pressure27(10,10,10)", {"ilu.variant": "ilut", "ilu.droptol": "1e-3",
                                                       "ilu.lfill": "5"}, 5, 102),
    ("c3_cutcell_16", "cutcell(16,16,16)", {}, 20, 103),
    ("ref_poisson2d_32", "poisson2d(32,32)", {}, 10, 104),
]

SOLVES = {
    "poisson2d(32,32)|gs": ("poisson2d(32,32)", {"krylov.tol": "1e-8"}),
    "poisson2d(32,32)|ilu55": ("poisson2d(32,32)", {"krylov.tol": "1e-8", "smoother.kind": "ilu",
                                                    "trisolve.m_lower": "5", "trisolve.m_upper": "5"}),
    "poisson3d(24,24,24)|ilu55|pmis": ("poisson3d(24,24,24)", {"krylov.tol": "1e-8", "smoother.kind": "ilu",
                                                               "trisolve.m_lower": "5", "trisolve.m_upper": "5",
                                                               "amg.coarsening": "pmis"}),
}


def main():
    ref = oracle.Ref()
    for name, spec, kv, m, seed in CASES:
        A = ilug.Matrix.generate(spec)
        Acsr = A.csr()
        Ar = ref.mat(*Acsr)
        assert all(np.array_equal(x, y) for x, y in zip(Acsr, ref.arrays(Ar)))
        f = ref.ilu(Ar, ref.cfg(kv))
        fs = ref.scale(f, "row")
        L, _, _, _ = ref.factors_arrays(f)
        b = ref.random_uniform(A.rows, seed)
        np.savez_compressed(
            os.path.join(HERE, name + ".npz"),
            spec=np.array(spec), kv_keys=np.array(list(kv.keys()), dtype=str),
            kv_vals=np.array(list(kv.values()), dtype=str), m=np.array(m), b=b,
            A_sha=np.array(hashlib.sha256(b"".join(a.tobytes() for a in Acsr)).hexdigest()),
            x_upper=ref.richardson_upper_scaled(fs, b, m),
            y_lower=ref.richardson_lower(ref.mat(*L), b, m),
            x_upper_direct=ref.solve_upper_scaled_direct(fs, b),
        )
        print("wrote", name)
    counts = {}
    for key, (spec, kv) in SOLVES.items():
        out = ref.run_solve(ilug.Matrix.generate(spec).csr(), kv)
        counts[key] = {"spec": spec, "kv": kv, "iterations": int(out["iterations"]),
                       "final_relres": float(out["final_relres"])}
    with open(os.path.join(HERE, "solve_counts.json"), "w") as fh:
        json.dump(counts, fh, indent=1, sort_keys=True)
    print("wrote solve_counts.json", counts)


if __name__ == "__main__":
    main()
