# C2 run_solve setup traces, repeated (setup-time variance diagnosis; not a test)
mkdir -p gpurun_out
for r in 1 2 3; do
  ILUG_DEFER_FREE=${DEFER:-1} timeout 600 python tools/probe_c2_setup.py > gpurun_out/setup_trace_$r.txt 2>&1
  grep "run_solve wall" gpurun_out/setup_trace_$r.txt
done
