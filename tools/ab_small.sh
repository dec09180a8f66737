#!/bin/bash
# small-config step times (two streams + serial split) and the parity tests touching the sketch-space sweeps
out=gpurun_out/ab_small.log; : > $out
for c in c0 c4 c2 c1 c3; do
  echo "== $c" >> $out
  timeout 300 python tools/quick_time.py $c 20 2>&1 | grep -E "ms/step" >> $out
  timeout 300 python tools/quick_time.py $c 20 serial 2>&1 | grep -E "ms/step|us/launch" >> $out
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_methods.py tests/test_gpu_sharded.py -q -x -p no:cacheprovider 2>&1 | tail -3 >> $out
timeout 1200 python -m pytest tests/test_gpu_golden.py -q -x -p no:cacheprovider -k "c0 or c2 or c4 or ex63" 2>&1 | tail -3 >> $out
