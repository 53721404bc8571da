# per-role wait profile of prefill v10 (trace build), then parity + timing on the normal build
mkdir -p gpurun_out
rm -f gpurun_out/v10_trace.log
make -s -C paper_2504_15720_b200/csrc clean >/dev/null; make -s -C paper_2504_15720_b200/csrc SKV_EXTRA=-DSKV_PF_TRACE > /dev/null 2>&1
for a in "4 16384 2048" "8 2048 512"; do
SEAKV_PREFILL_V=${TV:-10} SKV_TRACE=1 timeout 60 python scripts/prefill_trace.py $a >> gpurun_out/v10_trace.log 2>&1
done
make -s -C paper_2504_15720_b200/csrc clean >/dev/null; make -s -C paper_2504_15720_b200/csrc > /dev/null 2>&1
VERS="${VERS:-10}" bash scripts/v10run.sh
