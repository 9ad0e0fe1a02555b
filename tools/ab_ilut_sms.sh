# C2 run_solve setup vs the SMs the device ILUT's persistent grid may occupy
# (the rest stay free for the concurrent AMG setup; ILUG_ILUT_SMS A/B; not a test)
mkdir -p gpurun_out
for r in 1 2; do
  for v in ${SMS:-148 136 124}; do
    ILUG_ILUT_SMS=$v timeout 600 python tools/probe_c2_setup.py > gpurun_out/ilut_sms_${v}_$r.txt 2>&1
    echo "sms=$v $(grep 'run_solve wall' gpurun_out/ilut_sms_${v}_$r.txt) $(grep 'ilut-device factor kernel' gpurun_out/ilut_sms_${v}_$r.txt | tail -1)"
  done
done
