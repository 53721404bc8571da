# A/B of the v10 softmax paths (SKV_PREFILL_DBG=4: classic max-first softmax) + parity tests
mkdir -p gpurun_out; rm -f gpurun_out/v10ab.log
timeout 200 python -m pytest tests/test_gpu_prefill.py -x -q -p no:cacheprovider > gpurun_out/v10ab_tests.log 2>&1; echo "exit $?" >> gpurun_out/v10ab_tests.log
for a in "8 2048 512" "16 4096 1024" "4 16384 2048" "2 1024 512"; do
  for D in ${DBGS:-0 4}; do
    echo -n "dbg$D " >> gpurun_out/v10ab.log
    SKV_PREFILL_DBG=$D timeout 60 python scripts/prefill_probe.py $a >> gpurun_out/v10ab.log 2>&1
  done
done
nvidia-smi --query-gpu=clocks.sm,clocks_throttle_reasons.active --format=csv >> gpurun_out/v10ab.log
