"""Summarise an ncu report (raw page) into the JSON/markdown kept under profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/<name> [--bytes-per-launch B]

Writes <name>.json (per-launch metrics) and, when --bytes-per-launch is given,
profiles/u_sweep_traffic.json (dram bytes per launch, read by bench.py for
the roofline 'traffic' field)."""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "launch__waves_per_multiprocessor",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    bpl = None
    if "--bytes-per-launch" in sys.argv:
        bpl = float(sys.argv[sys.argv.index("--bytes-per-launch") + 1])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = r[i] + (f" {units[i]}" if units[i] else "")
        rb = float(r[hdr.index("dram__bytes_read.sum")]) * SCALE.get(units[hdr.index("dram__bytes_read.sum")], 1)
        wb = float(r[hdr.index("dram__bytes_write.sum")]) * SCALE.get(units[hdr.index("dram__bytes_write.sum")], 1)
        t = float(r[hdr.index("gpu__time_duration.sum")]) * SCALE.get(units[hdr.index("gpu__time_duration.sum")], 1)
        d["dram_bytes_total"] = rb + wb
        d["duration_s"] = t
        if bpl:
            d["algorithmic_bytes"] = bpl
            d["traffic_over_algorithmic"] = (rb + wb) / bpl
        launches.append(d)
    with open(out + ".json", "w") as fh:
        json.dump({"report": rep, "launches": launches}, fh, indent=1)
    if bpl:
        avg = sum(l["dram_bytes_total"] for l in launches) / len(launches)
        with open("profiles/u_sweep_traffic.json", "w") as fh:
            json.dump({"source": out + ".json", "dram_bytes_per_launch": avg, "algorithmic_bytes_per_launch": bpl,
                       "ratio": avg / bpl}, fh, indent=1)
    for l in launches:
        print(json.dumps(l))


if __name__ == "__main__":
    main()
