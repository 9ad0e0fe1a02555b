# run_solve setup with the device hierarchy built from the device AMG setup's
# own A_k/P_k/R_k copies vs re-uploaded from the host (ILUG_KEEP_DEVICE_LEVELS A/B); not a test
mkdir -p gpurun_out
for r in $(seq 1 ${REPS:-2}); do
  for v in 1 0; do
    ILUG_KEEP_DEVICE_LEVELS=$v timeout 600 python tools/probe_c2_setup.py > gpurun_out/keepdev_${v}_$r.txt 2>&1
    echo "C2 keep=$v $(grep 'run_solve wall' gpurun_out/keepdev_${v}_$r.txt)"
  done
done
for v in 1 0; do
  ILUG_KEEP_DEVICE_LEVELS=$v ILUG_TRACE_SETUP=1 timeout 900 python tools/run_c4.py "poisson3d(465,465,465)" richardson > gpurun_out/keepdev_c4_$v.txt 2>&1
  echo "C4 keep=$v $(tail -1 gpurun_out/keepdev_c4_$v.txt | cut -c1-400)"
done
