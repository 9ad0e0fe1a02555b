"""Host factorisation wall times (ILU(0), ILUT(1e-3,5)) for one matrix; not a test."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "pressure27(256,256,256)"
A = ilug.Matrix.generate(spec)
kv = {"ilu.droptol": "1e-3", "ilu.lfill": "5"}
for var in ("ilu0", "ilut"):
    t = time.time()
    L, U = ilug.ilu_factorize(A, ilug.Config().update(dict(kv, **{"ilu.variant": var})))
    print(f"{spec} {var} host {time.time() - t:.2f}s nnz(L)={L.nnz} nnz(U)={U.nnz}", flush=True)
