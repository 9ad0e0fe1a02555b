mkdir -p gpurun_out
for sg in 1024 8192 1024 8192; do
  ILUG_SELL_SIGMA=$sg NCU_REPS=3 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv -k regex:k_rowdot --kernel-name-base demangled python tools/ncu_targets.py step > gpurun_out/sig_$sg.csv 2>/dev/null
  echo "sigma $sg"; python - "$sg" <<'PY'
import csv,sys,collections
rows=[r for r in csv.reader(open(f"gpurun_out/sig_{sys.argv[1]}.csv")) if len(r)>10]
hdr=rows[0]; rows=rows[1:]
ki=hdr.index("Kernel Name"); mi=hdr.index("Metric Name"); vi=hdr.index("Metric Value"); ii=hdr.index("ID")
d=collections.OrderedDict()
for r in rows: d.setdefault(r[ii],{"k":r[ki]})[r[mi]]=r[vi]
L=list(d.values())[-9:]
tot=0
for e in L:
    t=float(e["gpu__time_duration.sum"].replace(",",""))
    tot+=t
    print(f"  {e['k'][:60]:60s} {t:9.1f}  rd {e['dram__bytes_read.sum']} wr {e['dram__bytes_write.sum']}")
print("  total", tot)
PY
done
