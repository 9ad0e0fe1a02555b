# C2 run_solve setup: the device ILUT's warps retire after QUOTA rows (their
# slots go to the higher-priority AMG/builder streams) vs a persistent grid
# (ILUG_ILUT_QUOTA=0); ILUT alone first (probe_ilut), then run_solve; not a test
mkdir -p gpurun_out
for r in 1 2 3; do
  for v in ${QUOTAS:-256 0}; do
    ILUG_ILUT_QUOTA=$v timeout 600 python tools/probe_c2_setup.py > gpurun_out/ilut_quota_${v}_$r.txt 2>&1
    echo "quota=$v $(grep 'run_solve wall' gpurun_out/ilut_quota_${v}_$r.txt) $(grep 'ilut-device factor kernel' gpurun_out/ilut_quota_${v}_$r.txt | tail -1)"
  done
done
