#!/bin/bash
# ping-pong prefill vs the one-tile kernel (SKV_PREFILL_PP=0), diagnostic builds, trace
for a in "8 2048 512" "4 16384 2048"; do
  echo -n "pp "; timeout 60 python scripts/prefill_probe.py $a 10
  echo -n "old "; SKV_PREFILL_PP=0 timeout 60 python scripts/prefill_probe.py $a 10
  for B in $BS; do echo -n "$B "; SKV_LIB_PATH=scripts/ab/libseakv_$B.so timeout 60 python scripts/prefill_probe.py $a 10; done
  echo -n "trace $a "; SKV_LIB_PATH=scripts/ab/libseakv_tr.so SKV_TRACE=1 timeout 60 python scripts/prefill_trace.py $a
done
