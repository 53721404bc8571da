# decode schedule knobs on the small config-1 launches (13B-only layers and the 7B+13B launch)
mkdir -p gpurun_out; rm -f gpurun_out/sweep_small.log
for c in 6 8 12; do for n in 1 2 3; do
  for a in "13b 520 32" "config1 520 32"; do
    echo "chunk $c ncut $n $(SKV_CHUNK_X4=$c SKV_NCUT_X4=$n timeout 60 python scripts/decode_probe.py $a 0 | tr -d '\n')" >> gpurun_out/sweep_small.log
  done
done; done
