#!/bin/bash
out=gpurun_out/ab_csr.log; : > $out
for v in 1 0; do
  echo "== SYLV_CSR_WINDOW=$v" >> $out
  SYLV_CSR_WINDOW=$v timeout 300 python tools/quick_time.py c4 20 serial 2>&1 | grep -E "pass1|pass2|ms/step|sketch" >> $out
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -x -p no:cacheprovider -k "csr" 2>&1 | tail -3 >> $out
