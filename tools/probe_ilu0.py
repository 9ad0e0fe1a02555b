"""Host vs device ILU(0) wall time on one matrix (setup-phase probe; not a test)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "pressure27(256,256,256)"
A = ilug.Matrix.generate(spec)
cfg = ilug.Config()
ilug.ilu_factorize_device(ilug.Matrix.generate("poisson3d(8,8,8)"), cfg)  # context + module load
t = time.time()
Ld, Ud = ilug.ilu_factorize_device(A, cfg)
td = time.time() - t
t = time.time()
Lh, Uh = ilug.ilu_factorize(A, cfg)
th = time.time() - t
same = all(np.array_equal(a.csr()[2].view(np.int64), b.csr()[2].view(np.int64)) for a, b in ((Ld, Lh), (Ud, Uh)))
print(f"{spec} n={A.rows} ilu0 device {td:.2f}s host {th:.2f}s bitwise={same}", flush=True)
