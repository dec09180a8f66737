timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -o faulthandler_timeout=300 -k "fused" > gpurun_out/pt.log 2>&1; echo tests $? >> gpurun_out/pt.log
SYLV_FUSED=1 timeout 300 python tools/quick_time.py c3 20 serial 2>&1 | grep -E "pass1:|pass2:" > gpurun_out/fused2.log
SYLV_FUSED=1 timeout 300 python tools/quick_time.py c3 20 2>&1 | grep -E "ms/step" >> gpurun_out/fused2.log
timeout 300 python tools/quick_time.py c3 20 2>&1 | grep -E "ms/step" >> gpurun_out/fused2.log
