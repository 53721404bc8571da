#!/bin/bash
# prefill probe: default build vs scripts/ab/libseakv_$B.so at the four probe shapes (+ head dims DS)
for D in ${DS:-128}; do
  for args in "8 2048 512" "16 4096 1024" "4 16384 2048" "2 1024 512"; do
    echo -n "A "; python scripts/prefill_probe.py $args 10 $D
    echo -n "B "; SKV_LIB_PATH=scripts/ab/libseakv_$B.so python scripts/prefill_probe.py $args 10 $D
  done
done
