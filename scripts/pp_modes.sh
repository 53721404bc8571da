#!/bin/bash
# prefill kernels for head dim 128 by SKV_PREFILL_PP mode (0 one-tile, 1 ping-pong, 2 ping-pong with
# two softmax warps per row set), REPS alternating runs at the probe shapes
for a in ${SHAPES:-"8 2048 512" "4 16384 2048"}; do
  for r in $(seq ${REPS:-3}); do
    for M in ${MODES:-0 1 2}; do
      echo -n "pp$M $a "; SKV_PREFILL_PP=$M timeout 60 python scripts/prefill_probe.py $a 10 | python3 -c "import json,sys; print(round(json.load(sys.stdin)['tflops'],1))"
    done
  done
done
