#!/bin/bash
# repeated alternating A/B of prefill builds (median of REPS runs each) at two shapes
for a in "8 2048 512" "4 16384 2048"; do
  for r in $(seq ${REPS:-3}); do
    echo -n "old $a "; SKV_PREFILL_PP=0 timeout 60 python scripts/prefill_probe.py $a 10 | python3 -c "import json,sys; print(round(json.load(sys.stdin)['tflops'],1))"
    for B in $BS; do echo -n "$B $a "; SKV_LIB_PATH=scripts/ab/libseakv_$B.so timeout 60 python scripts/prefill_probe.py $a 10 | python3 -c "import json,sys; print(round(json.load(sys.stdin)['tflops'],1))"; done
  done
done
