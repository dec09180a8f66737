set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo tests $?
timeout 600 python tools/quick_time.py c3 10 serial > gpurun_out/qt.log 2>&1; echo qt $?
timeout 600 python tools/ttt.py c0 >> gpurun_out/qt.log 2>&1
