"""A/B probe of the wavefront (fused multi-sweep) path vs the per-sweep kernels
(not a test, not the bench).

    python tools/probe_wave.py [SPEC] [ilu0|ilut]

Times sweep_upper / sweep_lower with m = 5 (1 scale pass + 4 sweeps) and the
fused-kernel entry for several grid sizes, CUDA events over 20 launches each.
GB/s are "effective": 4 sweeps' algorithmic bytes / time."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
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
out = {k: torch.empty_like(b) for k in ("0", "1")}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


F = {}
for wave in ("0", "1"):
    os.environ["ILUG_WAVEFRONT"] = wave
    F[wave] = ilug.Factors.from_csr(n, Lc, Uc, scaling="row")
    print(f"wave={wave} plans={F[wave].wave()}", flush=True)
st = F["0"].stats()
bytes_sweep = {"U": 12 * st["nnz_Us"] + 28 * n + 4, "L": 12 * st["nnz_Ls"] + 28 * n + 4}
VARIANTS = [{}, {}, {"ILUG_WAVE_L2_MB": "32"}, {"ILUG_WAVE_L2_MB": "128"}, {"ILUG_WAVE_HINTS": "1"},
            {"ILUG_WAVE_HINTS": "1", "ILUG_WAVE_L2_MB": "128"}, {"ILUG_WAVE_CTAS_PER_SM": "16"},
            {"ILUG_WAVE_CTAS_PER_SM": "4"}]
for var in VARIANTS:
    for k in ("ILUG_WAVE_L2_MB", "ILUG_WAVE_HINTS", "ILUG_WAVE_CTAS_PER_SM"):
        os.environ.pop(k, None)
    os.environ.update(var)
    for name, attr in (("U", "sweep_upper"), ("L", "sweep_lower")):
        row = []
        for wave in ("0", "1"):
            fn = getattr(F[wave], attr)
            ms = timeit(lambda: fn(b, out[wave], 5))
            gbs = 4 * bytes_sweep[name] / (ms * 1e-3) / 1e9
            row.append(f"wave={wave}: {ms * 1e3:8.1f} us ({gbs:7.1f} eff GB/s)")
        same = torch.equal(out["0"], out["1"])
        w = F["1"].wave()
        print(f"{str(var):48s} {name} m=5  " + "  ".join(row) + f"  bitwise={same} waits={w['waits']}"
              f" stalled={w['stalled']}", flush=True)
for k in ("ILUG_WAVE_L2_MB", "ILUG_WAVE_HINTS", "ILUG_WAVE_CTAS_PER_SM"):
    os.environ.pop(k, None)
print("stalled:", F["1"].wave()["stalled"])

# the smoother (L phase + U phase fused) end to end
for wave in ("0", "1"):
    os.environ["ILUG_WAVEFRONT"] = wave
    t = time.time()
    S = ilug.Smoother(A, ilug.Config().update(kv))
    x = torch.zeros_like(b)
    ms = timeit(lambda: S.ilu_sweep(b, x))
    print(f"smoother wave={wave}: ilu_sweep {ms * 1e3:8.1f} us (build {time.time() - t:.1f}s) {S.wave()}",
          flush=True)
    del S
