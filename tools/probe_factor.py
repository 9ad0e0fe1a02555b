"""Host vs device factorisation wall times (ILU(0), ILUT(1e-3,5)) for one matrix,
and whether the two agree bitwise; not a test.

    python tools/probe_factor.py [SPEC]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "pressure27(256,256,256)"
A = ilug.Matrix.generate(spec)
kv = {"ilu.droptol": "1e-3", "ilu.lfill": "5"}
for var in ("ilu0", "ilut"):
    cfg = ilug.Config().update(dict(kv, **{"ilu.variant": var}))
    if ilug.device_count() > 0:
        ilug.ilu_factorize_device(A, cfg)  # warm-up (module load, first allocations)
    t = time.time()
    Lh, Uh = ilug.ilu_factorize(A, cfg)
    th = time.time() - t
    msg = f"{spec} {var} host {th:.2f}s nnz(L)={Lh.nnz} nnz(U)={Uh.nnz}"
    if ilug.device_count() > 0:
        t = time.time()
        Ld, Ud = ilug.ilu_factorize_device(A, cfg)
        td = time.time() - t
        same = all(np.array_equal(d, h) for M, N in ((Ld, Lh), (Ud, Uh)) for d, h in zip(M.csr(), N.csr()))
        msg += f" device {td:.2f}s bitwise={same}"
    print(msg, flush=True)
