#!/bin/bash
# per-role wait profile (trace builds) at the short and long probe shapes + diagnostic timings
for a in "8 2048 512" "4 16384 2048"; do
  for B in tr trns; do echo -n "$B $a "; SKV_LIB_PATH=scripts/ab/libseakv_$B.so SKV_TRACE=1 timeout 60 python scripts/prefill_trace.py $a; done
  for B in ns nomufu; do echo -n "$B "; SKV_LIB_PATH=scripts/ab/libseakv_$B.so timeout 60 python scripts/prefill_probe.py $a 10; done
  echo -n "A "; timeout 60 python scripts/prefill_probe.py $a 10
done
