# Round-end measurement set (one GPU): bench without ncu first, then the ncu
# launch list of the same command and full captures of the U and L sweeps.
set -e
mkdir -p gpurun_out/ncu
timeout 900 python bench.py --steps 2 --warmup 1 --no-tts --no-cpu-baseline > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
    python bench.py --steps 2 --warmup 1 --no-tts --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_final.csv gpurun_out/prof_bench.json > gpurun_out/launches_final_summary.txt
for w in u l; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:EpiResidual -c 1 -f -o gpurun_out/ncu/final_$w python tools/ncu_targets.py $w > gpurun_out/ncu/final_$w.log 2>&1
done
tail -3 gpurun_out/launches_final_summary.txt
