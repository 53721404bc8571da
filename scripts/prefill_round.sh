# prefill evidence: probe of the default kernel vs v9 at the four probe sizes + one ncu --set full capture
mkdir -p gpurun_out
rm -f gpurun_out/prefill_probe.log
for a in "8 2048 512" "16 4096 1024" "4 16384 2048" "2 1024 512"; do
  for V in ${VERS:-10 9}; do
    echo -n "v$V " >> gpurun_out/prefill_probe.log
    SEAKV_PREFILL_V=$V timeout 60 python scripts/prefill_probe.py $a >> gpurun_out/prefill_probe.log 2>&1
  done
done
nvidia-smi --query-gpu=clocks.sm,clocks_throttle_reasons.active --format=csv >> gpurun_out/prefill_probe.log
if [ -n "$PROF" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_kernel_v -s 2 -c 1 \
  -o gpurun_out/prof_prefill_v10 -f python scripts/prefill_probe.py 4 16384 2048 3 > gpurun_out/prof_prefill_v10.log 2>&1
fi
