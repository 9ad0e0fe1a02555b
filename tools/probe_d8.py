"""SELL-D8 (dictionary-coded columns) vs the int32 column stream on the
bench's C2 smoother step: two smoothers built in one process (ILUG_SELL_D8
read at build time), interleaved timings, bitwise check (not a test).

    python tools/probe_d8.py [SPEC]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "pressure27(256,256,256)"
kv = {"smoother.kind": "ilu", "ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5",
      "trisolve.m_lower": "5", "trisolve.m_upper": "5", "smoother.sweeps": "1"}
torch.cuda.set_device(0)
A = ilug.Matrix.generate(spec)
n = A.rows
S = {}
for name, env in (("d8", "1"), ("i32", "0")):
    os.environ["ILUG_SELL_D8"] = env
    t = time.time()
    S[name] = ilug.Smoother(A, ilug.Config().update(kv))
    print(f"build {name} {time.time() - t:.1f}s", flush=True)
b = torch.rand(n, dtype=torch.float64, device="cuda")
xin = torch.rand(n, dtype=torch.float64, device="cuda")
out = torch.empty_like(b)
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


res = {}
for name, s in S.items():
    x = xin.clone()
    s.smooth(b, x)
    torch.cuda.synchronize()
    res[name] = x.cpu().numpy()
print("bitwise", bool(np.array_equal(res["d8"].view(np.int64), res["i32"].view(np.int64))), flush=True)
for rnd in range(3):
    for name, s in S.items():
        x = torch.zeros_like(b)
        step = timeit(lambda: s.smooth(b, x))
        once = lambda w: ilug._check(ilug.lib.ilug_smoother_sweep_once(s.h, w, xin.data_ptr(), b.data_ptr(),
                                                                        out.data_ptr(), st.cuda_stream))
        u, lo = timeit(lambda: once(1)), timeit(lambda: once(0))
        print(f"round {rnd} {name:4s} step {step:6.3f} ms ({28.47e9 / (step * 1e-3) / 1e9:6.0f} GB/s alg)  "
              f"U {u * 1e3:6.1f} us  L {lo * 1e3:6.1f} us", flush=True)
