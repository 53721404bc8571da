#!/bin/bash
# ncu evidence (single GPU): launch list of a short bench + one full capture of the top kernel.
mkdir -p gpurun_out
REQ=${REQ:-64}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-600} --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --requests $REQ --no-cpu-baseline \
  > gpurun_out/ncu_launches_stdout.log 2>&1
echo "launch list exit $?" >> gpurun_out/ncu_launches_stdout.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-decode_kernel} -s ${SKIP:-3} -c 1 \
  -o gpurun_out/prof_${TAG:-decode} python bench.py --steps 1 --warmup 1 --requests ${REQF:-32} --no-cpu-baseline \
  > gpurun_out/ncu_full_stdout.log 2>&1
echo "full exit $?" >> gpurun_out/ncu_full_stdout.log
