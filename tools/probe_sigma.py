"""SELL-C-sigma window A/B on the bench's smoother (not a test): for each sigma,
build the C2 smoother and time the bare L and U sweeps and the full step
(CUDA events, same process). The factorisation runs once (host ILUT); each
sigma only re-packs.

    python tools/probe_sigma.py [sigmas]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_09512_b200 as ilug  # noqa: E402

sigmas = (sys.argv[1] if len(sys.argv) > 1 else "1,256,512,1024").split(",")
kv = {"smoother.kind": "ilu", "ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5",
      "trisolve.m_lower": "5", "trisolve.m_upper": "5", "smoother.sweeps": "1"}
A = ilug.Matrix.generate("pressure27(256,256,256)")
n = A.rows
b = torch.rand(n, dtype=torch.float64, device="cuda")
xin = torch.rand(n, dtype=torch.float64, device="cuda")
out = torch.empty_like(b)
x = torch.zeros_like(b)
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timeit(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for sg in sigmas:
    os.environ["ILUG_SELL_SIGMA"] = sg
    t = time.time()
    S = ilug.Smoother(A, ilug.Config().update(kv))
    v = [C.c_longlong() for _ in range(5)]
    ilug._check(ilug.lib.ilug_smoother_stats(S.h, *[C.byref(q) for q in v]))
    _, _, nl, nu, pad = (q.value for q in v)
    once = lambda w: ilug._check(ilug.lib.ilug_smoother_sweep_once(S.h, w, xin.data_ptr(), b.data_ptr(),
                                                                    out.data_ptr(), st.cuda_stream))
    u, lo = timeit(lambda: once(1)), timeit(lambda: once(0))
    step = timeit(lambda: S.smooth(b, x))
    gb = lambda nnz, ms: (12 * nnz + 28 * n + 4) / (ms * 1e-3) / 1e9
    print(f"sigma={sg:5s} padU={pad / nu - 1:.3f} U {u * 1e3:6.1f} us {gb(nu, u):6.0f} GB/s  "
          f"L {lo * 1e3:6.1f} us {gb(nl, lo):6.0f} GB/s  step {step:.3f} ms  (build {time.time() - t:.0f}s)",
          flush=True)
    del S
