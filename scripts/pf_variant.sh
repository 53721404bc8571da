# parity tests + probe of one prefill variant: V=<n> bash scripts/pf_variant.sh
mkdir -p gpurun_out; rm -f gpurun_out/pfv.log
SEAKV_PREFILL_V=$V timeout 200 python -m pytest tests/test_gpu_prefill.py -x -q -p no:cacheprovider > gpurun_out/pfv_tests.log 2>&1; echo "exit $?" >> gpurun_out/pfv_tests.log
for a in "8 2048 512" "16 4096 1024" "4 16384 2048" "2 1024 512"; do
  for VV in $V ${REF:-10}; do
    echo -n "v$VV " >> gpurun_out/pfv.log
    SEAKV_PREFILL_V=$VV timeout 60 python scripts/prefill_probe.py $a >> gpurun_out/pfv.log 2>&1
  done
done
