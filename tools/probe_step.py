"""Interleaved A/B of kernel variants on the bench's smoother step (not a test,
not the bench): one C2 smoother, then rounds of {variant: env} timings in the
same process, so box-to-box noise cancels.

    python tools/probe_step.py [SPEC] VAR=VAL[,VAR=VAL] [VAR=VAL ...]

Each argument after SPEC is one variant (comma-separated env assignments;
"base" = no change). Prints ms per smoother step (m_L = m_U = 5) and per bare
U sweep (CUDA events, 30 launches) for every round."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2111_09512_b200 as ilug  # noqa: E402

args = sys.argv[1:]
spec = args.pop(0) if args and "(" in args[0] else "pressure27(256,256,256)"
variants = args or ["base", "ILUG_PDL=1"]
kv = {"smoother.kind": "ilu", "ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5",
      "trisolve.m_lower": "5", "trisolve.m_upper": "5", "smoother.sweeps": "1"}
torch.cuda.set_device(0)
t = time.time()
A = ilug.Matrix.generate(spec)
S = ilug.Smoother(A, ilug.Config().update(kv))
n = A.rows
print(f"setup {time.time() - t:.1f}s n={n}", flush=True)
b = torch.rand(n, dtype=torch.float64, device="cuda")
x = torch.zeros_like(b)
xin = torch.rand(n, dtype=torch.float64, device="cuda")
out = torch.empty_like(b)
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def once(which):
    ilug._check(ilug.lib.ilug_smoother_sweep_once(S.h, which, xin.data_ptr(), b.data_ptr(), out.data_ptr(),
                                                  st.cuda_stream))


keys = set()
for v in variants:
    if v != "base":
        keys |= {kv_.split("=")[0] for kv_ in v.split(",")}
for rnd in range(3):
    for v in variants:
        for k in keys:
            os.environ.pop(k, None)
        if v != "base":
            for kv_ in v.split(","):
                k, val = kv_.split("=", 1)
                os.environ[k] = val
        step = timeit(lambda: S.smooth(b, x), 30)
        u = timeit(lambda: once(1), 30)
        lo = timeit(lambda: once(0), 30)
        print(f"round {rnd} {v:32s} step {step:7.3f} ms  U sweep {u * 1e3:7.1f} us  L sweep {lo * 1e3:7.1f} us",
              flush=True)
