"""Host AMG setup phase times (ILUG_TRACE_SETUP) for one matrix; not a test.

    python tools/probe_setup.py SPEC [key=value ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ILUG_TRACE_SETUP"] = "1"
import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1]
kv = {"amg.coarsening": "pmis"}
kv.update(dict(a.split("=", 1) for a in sys.argv[2:]))
t = time.time()
A = ilug.Matrix.generate(spec)
print(f"generate {time.time() - t:.2f}s n={A.rows} nnz={A.nnz}", file=sys.stderr, flush=True)
t = time.time()
H = ilug.Hierarchy(A, ilug.Config().update(kv), host_only=True)
print(f"amg host total {time.time() - t:.2f}s levels={H.levels}", file=sys.stderr, flush=True)
