#!/bin/bash
# development call: compact (masked) SELL storage for uneven rows — CSR parity tests and c4 A/B
out=gpurun_out/dev6.log; : > $out
echo "== parity csr" >> $out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "csr" 2>&1 | tail -5 >> $out
for v in auto off; do
  if [ $v = off ]; then export SYLV_SELL_COMPACT=0; else unset SYLV_SELL_COMPACT; fi
  echo "== c4 $v serial" >> $out
  timeout 200 python tools/quick_time.py c4 20 serial 2>&1 | grep -E "pass1|ms/step" >> $out
  echo "== c4 $v" >> $out
  timeout 200 python tools/quick_time.py c4 40 2>&1 | grep -E "ms/step" >> $out
done
unset SYLV_SELL_COMPACT
echo "== forced compact on every CSR operator: parity csr" >> $out
SYLV_SELL_COMPACT=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "csr" 2>&1 | tail -3 >> $out
echo "== sharded/methods/fullsize/golden csr" >> $out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_methods.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "csr or c4 or ex6" 2>&1 | tail -3 >> $out
timeout 900 python -m pytest tests/test_gpu_golden.py -q -x -p no:cacheprovider -k "c4 or ex63 or nu0.1" 2>&1 | tail -3 >> $out
timeout 600 python bench.py --config c4 --no-cpu-baseline > gpurun_out/dev6_c4.json 2> gpurun_out/dev6_c4.err
cat $out
