# C2 run_solve setup with one shared device upload of A vs two (ILUG_SHARE_A A/B; not a test)
mkdir -p gpurun_out
for r in 1 2 3; do
  for v in 1 0; do
    ILUG_SHARE_A=$v timeout 600 python tools/probe_c2_setup.py > gpurun_out/share_a_${v}_$r.txt 2>&1
    echo "share_A=$v $(grep 'run_solve wall' gpurun_out/share_a_${v}_$r.txt)"
  done
done
