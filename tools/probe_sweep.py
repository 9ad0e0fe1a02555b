"""Kernel A/B probe for the sweep kernels (not a test, not the bench).

    python tools/probe_sweep.py [SPEC] [ilu0|ilut]

Builds the factors once on the host, then for each (ILUG_SELL_SIGMA,
ILUG_L2_HINTS) variant uploads/packs them and times the bare U and L sweep
kernels (CUDA events, 50 launches) — algorithmic GB/s per SURVEY.md §8d."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "pressure27(256,256,256)"
variant = sys.argv[2] if len(sys.argv) > 2 else "ilut"
kv = {"smoother.kind": "ilu", "ilu.variant": variant, "ilu.droptol": "1e-3", "ilu.lfill": "5",
      "trisolve.m_lower": "5", "trisolve.m_upper": "5", "smoother.sweeps": "1"}
torch.cuda.set_device(0)
t = time.time()
A = ilug.Matrix.generate(spec)
L, U = ilug.ilu_factorize(A, ilug.Config().update(kv))
Lc, Uc = L.csr(), U.csr()
n = A.rows
print(f"setup {time.time() - t:.1f}s n={n} nnzL={L.nnz} nnzU={U.nnz}", flush=True)
del L, U
b = torch.rand(n, dtype=torch.float64, device="cuda")
xin = torch.rand(n, dtype=torch.float64, device="cuda")
out = torch.empty_like(b)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for sigma in os.environ.get("PROBE_SIGMAS", "1024").split(","):
    os.environ["ILUG_SELL_SIGMA"] = sigma
    F = ilug.Factors.from_csr(n, Lc, Uc, scaling="row")
    st = F.stats()
    var = os.environ.get("PROBE_VAR", "ILUG_ROWDOT_BLOCK")  # the A/B knob to sweep
    for rep, hints in enumerate(os.environ.get("PROBE_BLOCKS", "256").split(",")):
        os.environ[var] = hints
        res = []
        for name, fn, nnz in (("U", F.sweep_upper, st["nnz_Us"]), ("L", F.sweep_lower, st["nnz_Ls"])):
            # m=2 = one scale/copy pass + one SpMV sweep; isolate the sweep by differencing m=3 - m=2
            for _ in range(3):
                fn(b, out, 3)
            torch.cuda.synchronize()
            ts = {}
            for m in (2, 6):
                e0.record()
                for _ in range(20):
                    fn(b, out, m)
                e1.record()
                torch.cuda.synchronize()
                ts[m] = e0.elapsed_time(e1) / 20
            ms = (ts[6] - ts[2]) / 4
            gbs = (12 * nnz + 28 * n + 4) / (ms * 1e-3) / 1e9
            res.append(f"{name}: {ms * 1e3:7.1f} us {gbs:7.1f} GB/s")
        print(f"sigma={sigma:5s} {var}={hints} padded_U={st['padded_Us'] / st['nnz_Us'] - 1:.3f}  " + "  ".join(res),
              flush=True)
    del F
