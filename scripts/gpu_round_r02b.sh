#!/bin/bash
# round-2 closing evidence: GPU tests, smoke, default bench, ping-pong prefill ncu capture + launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:prefill_pp -s 1 -c 1 -o gpurun_out/prof_pp_final -f python scripts/prefill_probe.py 4 16384 2048 2 > gpurun_out/prof_pp_final.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:prefill_pp -s 1 -c 1 -o gpurun_out/prof_pp_short -f python scripts/prefill_probe.py 8 2048 512 2 > gpurun_out/prof_pp_short.log 2>&1
