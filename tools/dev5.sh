#!/bin/bash
# development call: rotated slice map + wide fold — parity tests, c4 / c2 timing, SYLV_SELL_RING A/B
out=gpurun_out/dev5.log; : > $out
echo "== c4 serial" >> $out
timeout 200 python tools/quick_time.py c4 20 serial 2>&1 | grep -E "pass1|pass2|ms/step|sketch" >> $out
echo "== c4" >> $out
timeout 200 python tools/quick_time.py c4 40 2>&1 | grep -E "ms/step" >> $out
echo "== c2" >> $out
timeout 200 python tools/quick_time.py c2 40 2>&1 | grep -E "ms/step" >> $out
timeout 200 python tools/quick_time.py c2 40 serial 2>&1 | grep -E "ms/step|sketch" >> $out
echo "== parity + sketch pull" >> $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sketch_pull.py -q -x -p no:cacheprovider 2>&1 | tail -3 >> $out
echo "== sharded/methods/fullsize csr" >> $out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_methods.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "csr or c4 or ex6" 2>&1 | tail -3 >> $out
timeout 900 python -m pytest tests/test_gpu_golden.py -q -x -p no:cacheprovider -k "c4 or ex63 or nu0.1" 2>&1 | tail -3 >> $out
cat $out
