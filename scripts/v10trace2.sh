# per-role wait profile of prefill v10: normal and softmax-free (diagnostic) trace builds
mkdir -p gpurun_out; rm -f gpurun_out/v10_trace2.log
for X in "-DSKV_PF_TRACE" "-DSKV_PF_TRACE -DSKV_PF_NOSOFTMAX"; do
  make -s -C paper_2504_15720_b200/csrc clean >/dev/null; make -s -C paper_2504_15720_b200/csrc SKV_EXTRA="$X" > /dev/null 2>&1
  for a in "4 16384 2048"; do
    echo -n "[$X] " >> gpurun_out/v10_trace2.log
    SEAKV_PREFILL_V=10 SKV_TRACE=1 timeout 60 python scripts/prefill_trace.py $a >> gpurun_out/v10_trace2.log 2>&1
  done
done
make -s -C paper_2504_15720_b200/csrc clean >/dev/null; make -s -C paper_2504_15720_b200/csrc > /dev/null 2>&1
