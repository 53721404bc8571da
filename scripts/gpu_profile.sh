#!/bin/bash
# ncu evidence (single GPU), all under gpurun_out/:
#  1. launch list of a short full-size config-2 bench (per-kernel share of the step)
#  2. DRAM traffic of full-size decode launches (single-pass metrics: no 122 GB save/restore)
#  3. one --set full capture of the top kernel at reduced size
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-200} --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-graph ${BENCH_ARGS} \
  > gpurun_out/ncu_launches_stdout.log 2>&1
echo "launch list exit $?" >> gpurun_out/ncu_launches_stdout.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:decode_kernel -s 4 -c 3 --csv --log-file gpurun_out/decode_traffic.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-graph ${BENCH_ARGS} > gpurun_out/ncu_traffic_stdout.log 2>&1
echo "traffic exit $?" >> gpurun_out/ncu_traffic_stdout.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-decode_kernel} -s ${SKIP:-3} -c 1 \
  -o gpurun_out/prof_${TAG:-decode} python bench.py --steps 1 --warmup 1 --requests ${REQF:-32} --no-cpu-baseline --no-graph \
  ${BENCH_ARGS} > gpurun_out/ncu_full_stdout.log 2>&1
echo "full exit $?" >> gpurun_out/ncu_full_stdout.log
