mkdir -p gpurun_out
for v in "8 3" "6 4" "4 6"; do set -- $v
  touch paper_2504_15720_b200/csrc/skv_attn.cu paper_2504_15720_b200/csrc/skv_capi.cpp
  make -s -C paper_2504_15720_b200/csrc SKV_EXTRA="-DSKV_DEC_WARPS=$1 -DSKV_DEC_STAGES=$2" > /dev/null 2>&1
  echo "== warps $1 stages $2"
  for a in "config1 520 32" "13b 520 32" "config2s 2048 64" "config2s 2048 256" "13b 8192 4"; do timeout 100 python scripts/decode_probe.py $a 0 | tr -d '\n'; echo; done
done
