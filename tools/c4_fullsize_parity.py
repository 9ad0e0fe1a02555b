"""One-off evidence (not in the test suite: minutes of single-threaded
reference work): a BASELINE smoother step at FULL size — by default C4,
poisson3d(465^3), 100.5 M rows, ILU(0) row-scaled, m_L = m_U = 5 — on the
device (the distributed smoother's rank-local form at p = 1, i.e. the bench's
`--strong` step at N = 1) versus the reference library's ilu_smooth_sweep on
the same matrix built by the oracle-side generator. Prints one JSON line.

    python tools/c4_fullsize_parity.py [SPEC [scaling]]   (e.g. "cutcell(256,256,256)" row_col)"""
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_09512_b200 as ilug  # noqa: E402
from paper_2111_09512_b200 import dist as idist  # noqa: E402
from oracle import oracle  # noqa: E402

SPEC = sys.argv[1] if len(sys.argv) > 1 else "poisson3d(465,465,465)"
KV = {"smoother.kind": "ilu", "ilu.variant": "ilu0", "scaling": sys.argv[2] if len(sys.argv) > 2 else "row",
      "trisolve.mode": "richardson",
      "trisolve.m_lower": "5", "trisolve.m_upper": "5", "smoother.sweeps": "1"}
torch.cuda.set_device(0)
out = {"spec": SPEC, "scaling": KV["scaling"], "sell_d8": os.environ.get("ILUG_SELL_D8", "1")}
t = time.time()
A = ilug.Matrix.generate(SPEC)
n = A.rows
rows = idist.generate_rows(SPEC, 0, n)
plan = idist.Plan(rows, n, 1, 0)
comm = idist.Comm(1, 0, idist.unique_id())
plan.exchange(comm)
S = idist.Smoother(plan, comm, ilug.Config().update(KV))
rng = np.random.default_rng(465)
b, x0 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
bd, xd = torch.from_numpy(b).cuda(), torch.from_numpy(x0.copy()).cuda()
torch.cuda.synchronize()
out["device_setup_s"] = round(time.time() - t, 1)
S.smooth(bd, xd)
torch.cuda.synchronize()
got = xd.cpu().numpy()
del S, plan, rows
ref = oracle.Ref()
t = time.time()
Ar = ref.gen3d(SPEC)
rp, ci, v = A.csr()
h = lambda *a: hashlib.sha256(b"".join(np.ascontiguousarray(x).tobytes() for x in a)).hexdigest()
rrp, rci, rv = ref.arrays(Ar)
out["same_matrix"] = h(rp.astype(np.int64), ci.astype(np.int64), v) == h(rrp, rci, rv)
del rrp, rci, rv, rp, ci, v
st = ref.smoother(Ar, ref.cfg(KV))
out["reference_setup_s"] = round(time.time() - t, 1)
t = time.time()
want = ref.ilu_smooth_sweep(Ar, st, b, x0)
out["reference_step_s"] = round(time.time() - t, 1)
out["bitwise"] = bool(np.array_equal(got.view(np.int64), want.view(np.int64)))
out["max_abs_diff"] = float(np.abs(got - want).max())
print(json.dumps(out), flush=True)
