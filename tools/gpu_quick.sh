timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -o faulthandler_timeout=300 -k "r4" > gpurun_out/pt.log 2>&1; echo tests $? >> gpurun_out/pt.log
for i in 1 2; do timeout 300 python tools/quick_time.py c2 20 serial 2>&1 | grep -E "pass1:|pass2:" >> gpurun_out/occ6.log; done
timeout 300 python tools/quick_time.py c2 20 2>&1 | grep -E "ms/step" >> gpurun_out/occ6.log
