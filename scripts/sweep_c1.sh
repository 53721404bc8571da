#!/bin/bash
# config-1 decode schedule knobs in the bench's graph-replayed step (value = GB/s over the step)
for c in 6 3 12 100; do for n in -1 2 4 8 16; do
  if [ "$n" = "-1" ]; then unset SKV_NCUT_X4; else export SKV_NCUT_X4=$n; fi
  echo -n "chunk $c ncut $n "; SKV_CHUNK_X4=$c timeout 120 python bench.py --workload config1 --steps 10 --warmup 3 --no-prefill --no-cpu-baseline --no-faithful --no-parity 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'])"
done; done
