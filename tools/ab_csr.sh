#!/bin/bash
# A/B of the c4 CSR pass 1 variants (SELL-32 window / CSR-stream window / global gathers) and c2
out=gpurun_out/ab_csr.log; : > $out
for v in sell csrwin global; do
  case $v in
    sell) unset SYLV_SELL SYLV_CSR_WINDOW;;
    csrwin) export SYLV_SELL=0; unset SYLV_CSR_WINDOW;;
    global) export SYLV_CSR_WINDOW=0;;
  esac
  echo "== $v" >> $out
  timeout 300 python tools/quick_time.py c4 20 serial 2>&1 | grep -E "pass1|pass2|ms/step|sketch" >> $out
done
unset SYLV_SELL SYLV_CSR_WINDOW
echo "== c2" >> $out
timeout 300 python tools/quick_time.py c2 20 serial 2>&1 | grep -E "pass1|pass2|ms/step" >> $out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_methods.py -q -x -p no:cacheprovider -k "csr or r4" 2>&1 | tail -3 >> $out
