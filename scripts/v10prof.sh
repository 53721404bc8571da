mkdir -p gpurun_out
for V in 10 9; do
SEAKV_PREFILL_V=$V timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_kernel_v -s 2 -c 1 \
  -o gpurun_out/prof_pf_v$V python scripts/prefill_probe.py 4 16384 2048 3 > gpurun_out/prof_pf_v$V.log 2>&1
done
