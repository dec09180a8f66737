timeout 300 python tools/quick_time.py c3 10 serial > gpurun_out/qt.log 2>&1
timeout 300 python tools/quick_time.py c2 10 serial >> gpurun_out/qt.log 2>&1
