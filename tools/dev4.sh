#!/bin/bash
# development call: length-sorted SELL rows (ring kernel) — CSR parity tests and c4 timing
out=gpurun_out/dev4.log; : > $out
echo "== parity csr" >> $out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "csr" 2>&1 | tail -5 >> $out
echo "== c4 serial" >> $out
timeout 200 python tools/quick_time.py c4 20 serial 2>&1 | grep -E "pass1|pass2|ms/step|sketch" >> $out
echo "== c4" >> $out
timeout 200 python tools/quick_time.py c4 40 2>&1 | grep -E "ms/step" >> $out
echo "== sharded/methods/fullsize csr" >> $out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_methods.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "csr or c4 or ex6" 2>&1 | tail -3 >> $out
timeout 900 python -m pytest tests/test_gpu_golden.py -q -x -p no:cacheprovider -k "c4 or ex63 or nu0.1" 2>&1 | tail -3 >> $out
cat $out
