set -x
timeout 200 python tools/quick_time.py c2 10 serial > gpurun_out/qt.log 2>&1
timeout 200 python tools/quick_time.py c3 10 serial >> gpurun_out/qt.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "tma" -o faulthandler_timeout=200 > gpurun_out/gputest.log 2>&1; echo tests $?
