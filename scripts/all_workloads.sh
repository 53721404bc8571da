# every bench workload once (default K/W), one JSON line each, into gpurun_out/workloads.log
mkdir -p gpurun_out; rm -f gpurun_out/workloads.log
for w in config1 config2 config3 config4 config5 prefill; do
  echo "== $w" >> gpurun_out/workloads.log
  timeout 600 python bench.py --workload $w >> gpurun_out/workloads.log 2> gpurun_out/workloads_$w.err
  echo "exit $?" >> gpurun_out/workloads.log
done
