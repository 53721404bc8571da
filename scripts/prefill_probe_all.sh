#!/bin/bash
# prefill probe at the four round-1 probe shapes for each head dim
for D in ${DS:-128 64 256}; do
  for args in "8 2048 512" "16 4096 1024" "4 16384 2048" "2 1024 512"; do
    python scripts/prefill_probe.py $args 10 $D
  done
done
