#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py
# (run on the GPU box). Logs: gpurun_out/sanitizer/<tool>_<case>.log, summary on stdout.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sanitizer
CASES=${CASES:-"levelset_cta levelset_cta1 levelset_flags levelset_vflags ilu0_warp ilu0_thread ilut sweeps"}
TOOLS=${TOOLS:-"memcheck racecheck synccheck"}
for tool in $TOOLS; do
  for c in $CASES; do
    log=gpurun_out/sanitizer/${tool}_${c}.log
    timeout ${SAN_TIMEOUT:-420} /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 \
      python tools/sanitize_cases.py $c > $log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|OK \(bitwise' $log | tr '\n' ' ')"
  done
done
