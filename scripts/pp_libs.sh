#!/bin/bash
# default build vs scripts/ab/libseakv_$B.so builds, REPS alternating runs at the probe shapes
for a in ${SHAPES:-"8 2048 512" "4 16384 2048" "2 1024 512"}; do
  for r in $(seq ${REPS:-3}); do
    echo -n "new $a "; timeout 60 python scripts/prefill_probe.py $a 10 | python3 -c "import json,sys; print(round(json.load(sys.stdin)['tflops'],1))"
    for B in $BS; do echo -n "$B $a "; SKV_LIB_PATH=scripts/ab/libseakv_$B.so timeout 60 python scripts/prefill_probe.py $a 10 | python3 -c "import json,sys; print(round(json.load(sys.stdin)['tflops'],1))"; done
  done
done
