timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "csr" -o faulthandler_timeout=100 > gpurun_out/gputest.log 2>&1; echo tests $?
timeout 200 python tools/quick_time.py c4 10 serial > gpurun_out/qt.log 2>&1; echo qt $?
