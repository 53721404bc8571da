#!/bin/bash
# prefill probe at the four shapes for the default build (and optional A/B builds in $BS)
for args in "8 2048 512" "16 4096 1024" "4 16384 2048" "2 1024 512"; do
  echo -n "A "; timeout 60 python scripts/prefill_probe.py $args 10 ${D:-128}
  for B in $BS; do echo -n "$B "; SKV_LIB_PATH=scripts/ab/libseakv_$B.so timeout 60 python scripts/prefill_probe.py $args 10 ${D:-128}; done
done
nvidia-smi --query-gpu=clocks.sm,clocks_throttle_reasons.active --format=csv
