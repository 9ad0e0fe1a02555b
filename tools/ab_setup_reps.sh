# C2 run_solve setup repeated N times (default 6) on one box; prints each setup
# and any mid-setup deferred-free flush; not a test
mkdir -p gpurun_out
for r in $(seq 1 ${N:-6}); do
  timeout 600 python tools/probe_c2_setup.py > gpurun_out/setup_rep_$r.txt 2>&1
  echo "$(grep 'run_solve wall' gpurun_out/setup_rep_$r.txt) flushes=$(grep -c 'cap flush' gpurun_out/setup_rep_$r.txt)"
done
