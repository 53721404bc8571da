# diagnostic builds of prefill v10 (wrong results, timing only): MUFU off / tile math off
mkdir -p gpurun_out; rm -f gpurun_out/v10diag.log
for X in ${XS:-"" "-DSKV_PF_NOMUFU" "-DSKV_PF_NOSOFTMAX"}; do
  make -s -C paper_2504_15720_b200/csrc clean >/dev/null; make -s -C paper_2504_15720_b200/csrc SKV_EXTRA="$X" > /dev/null 2>&1
  for a in "8 2048 512" "4 16384 2048"; do
    echo -n "build[$X] " >> gpurun_out/v10diag.log
    timeout 60 python scripts/prefill_probe.py $a >> gpurun_out/v10diag.log 2>&1
  done
done
make -s -C paper_2504_15720_b200/csrc clean >/dev/null; make -s -C paper_2504_15720_b200/csrc > /dev/null 2>&1
