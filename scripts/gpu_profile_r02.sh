#!/bin/bash
# Round-2 evidence (one GPU), all under gpurun_out/:
#  1. config 3 bench lines: default pool, and a small pool where CacheFull / preemption fire
#  2. launch list of the default config-2 bench (graph path: grow + plan + decodes)
#  3. ncu --set full: decode on the mixed-head-dim config (reduced size), prefill d=64 / d=256,
#     the device-side decode-step grow kernel
mkdir -p gpurun_out
timeout 600 python bench.py --workload config3 > gpurun_out/b_config3.log 2>&1
timeout 600 python bench.py --workload config3 --pool-gb 25 --occupancy 0.95 > gpurun_out/b_config3_small.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_config2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-prefill --no-parity \
  > gpurun_out/ncu_launches_stdout.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 4 -c 1 \
  -o gpurun_out/prof_decode_config2d python bench.py --workload config2d --steps 1 --warmup 1 --requests 32 \
  --no-cpu-baseline --no-graph --no-prefill --no-parity > gpurun_out/ncu_full_decode_stdout.log 2>&1
for D in 64 256; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 2 -c 1 \
    -o gpurun_out/prof_prefill_d$D python scripts/prefill_probe.py 4 16384 2048 3 $D > gpurun_out/ncu_full_prefill_d$D.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:grow_kernel -s 20 -c 1 \
  -o gpurun_out/prof_grow python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-prefill --no-parity \
  > gpurun_out/ncu_full_grow.log 2>&1
echo done > gpurun_out/profile_done.txt
