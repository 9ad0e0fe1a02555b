"""One device ILUT(1e-3,5) factorisation of SPEC (ncu target); not a test.

    python tools/probe_ilut.py [SPEC] [repeats]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "pressure27(128,128,128)"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
A = ilug.Matrix.generate(spec)
cfg = ilug.Config().update({"ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5"})
for _ in range(reps):
    t = time.time()
    ilug.ilu_factorize_device(A, cfg)
    print(f"{spec} device ilut {time.time() - t:.3f}s", flush=True)
