"""Repeat one run_solve many times in one process and report any change in the
iteration count / final residual or any error (flakiness hunt; not a test).

    python tools/stress_solve.py SPEC N key=value ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1]
reps = int(sys.argv[2])
kv = dict(a.split("=", 1) for a in sys.argv[3:])
A = ilug.Matrix.generate(spec)
seen = {}
for i in range(reps):
    try:
        rep = ilug.run_solve(A, ilug.Config().update(kv))
        key = (rep["iterations"], rep["final_relres"])
    except ilug.IlugError as e:
        key = ("error", str(e)[:120])
    seen[key] = seen.get(key, 0) + 1
print(spec, kv, seen, flush=True)
