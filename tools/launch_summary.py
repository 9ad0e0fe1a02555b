"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv
--log-file F python bench.py ...`): per-kernel totals and the last smoother
step's nine launches with the U-sweep share (compared with the bench's own
share). Not a test.

    python tools/launch_summary.py gpurun_out/launches.csv [bench.json]"""
import collections
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
launches = [(r[ki], float(r[vi].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6,
                                                     "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6))
            for r in rows if r[mi] == "gpu__time_duration.sum"]
tot = collections.OrderedDict()
for k, ms in launches:
    c, t = tot.get(k, (0, 0.0))
    tot[k] = (c + 1, t + ms)
print("kernel | launches | total ms")
for k, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:110]} | {c} | {t:.3f}")
# the last smoother step: the last nine k_rowdot launches ending with the accumulating U sweep
idx = [i for i, (k, _) in enumerate(launches) if "EpiAcc" in k]
if idx:
    step = launches[idx[-1] - 8: idx[-1] + 1]
    print("\nlast smoother step (residual, 3 L, L+div, 3 U, U+acc):")
    for k, ms in step:
        print(f"{k[:100]} {ms:.4f} ms")
    s = sum(ms for _, ms in step)
    u3 = sum(ms for _, ms in step[5:8])
    line = f"step {s:.4f} ms; the three plain U sweeps {u3:.4f} ms = {100 * u3 / s:.1f}% of the step"
    if len(sys.argv) > 2:
        b = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
        r = b["roofline"]
        line += f" (bench: 3 x {r['ms_per_launch']:.3f} / {b['ms_per_step']:.3f} = " \
                f"{100 * 3 * r['ms_per_launch'] / b['ms_per_step']:.1f} %)"
    print(line)
