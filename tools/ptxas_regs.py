"""Registers / spills per kernel of one .cu file (reads `nvcc -Xptxas -v` output).

    python tools/ptxas_regs.py paper_2111_09512_b200/csrc/kernels/sell.cu [filter]"""
import re
import subprocess
import sys

src = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else ""
inc = src.split("/csrc/")[0] + "/../include" if "/csrc/" in src else "include"
cmd = ["nvcc", "-std=c++20", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "--fmad=false",
       "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-I" + inc, "-Xptxas", "-v", "-c", src, "-o", "/dev/null"]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
name = None
for line in out.splitlines():
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        name = subprocess.run(["cu++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name:
        spill = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        if flt in name:
            short = re.sub(r"ilug::\(anonymous namespace\)::", "", name)
            print(f"{int(m.group(1)):4d} regs  {short[:110]}")
        name = None
