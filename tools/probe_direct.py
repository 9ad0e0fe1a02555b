"""Direct (level-scheduled K5) triangular solves of the ILUT(1e-3,5) factors of
SPEC, timed with CUDA events (ncu target); not a test.

    python tools/probe_direct.py [SPEC] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "pressure27(128,128,128)"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
A = ilug.Matrix.generate(spec)
cfg = ilug.Config().update({"ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5"})
L, U = ilug.ilu_factorize_device(A, cfg)
f = ilug.Factors.from_csr(A.rows, L.csr(), U.csr(), scaling="row", direct=True)
st = f.stats()
b = torch.rand(A.rows, dtype=torch.float64, device="cuda")
y = torch.empty_like(b)
for _ in range(2):
    f.solve_lower(b, y)
    f.solve_upper(b, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
out = {}
for name, fn in (("lower", f.solve_lower), ("upper", f.solve_upper)):
    e0.record()
    for _ in range(reps):
        fn(b, y)
    e1.record()
    torch.cuda.synchronize()
    out[name] = e0.elapsed_time(e1) / reps
print(f"{spec}: levels L {st['levels_L']} U {st['levels_U']}  lower {out['lower']:.3f} ms  "
      f"upper {out['upper']:.3f} ms", flush=True)
