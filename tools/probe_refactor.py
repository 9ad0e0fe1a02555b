"""ILU(0) numeric refactorisation vs a fresh factor build at SPEC (wall times);
not a test.   python tools/probe_refactor.py [SPEC]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "pressure27(256,256,256)"
base, args = spec.split("(")
A1 = ilug.Matrix.generate(spec)
A2 = ilug.Matrix.generate(f"{base}({args[:-1]},7)")
cfg = ilug.Config()
t = time.time()
f = ilug.Factors.create(A1, cfg, scaling="row")
print(f"create {time.time() - t:.3f}s", flush=True)
for k in range(3):
    t = time.time()
    f.refactor(A2 if k % 2 == 0 else A1)
    print(f"refactor {time.time() - t:.3f}s", flush=True)
