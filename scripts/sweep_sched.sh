#!/bin/bash
# decode schedule knob sweep: SKV_CHUNK_X4 x SKV_NCUT_X4 over representative shapes
mkdir -p gpurun_out
for c in 0 4 6 16; do for n in 0 2 4 8 16; do
  for a in "config1 520 32" "13b 520 32" "config2s 2048 64" "config2s 2048 256" "13b 8192 4" "config2s 4096 16"; do
    echo "chunk $c ncut $n $(SKV_CHUNK_X4=$c SKV_NCUT_X4=$n python scripts/decode_probe.py $a 0 | tr -d '\n')"
  done
done; done
