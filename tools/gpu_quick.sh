set -x
timeout 600 python tools/quick_time.py c3 10 serial > gpurun_out/qt.log 2>&1; echo qt $?
timeout 300 python tools/quick_time.py c3 10 >> gpurun_out/qt.log 2>&1
for c in c2 c4 c1 c0; do timeout 300 python tools/quick_time.py $c 10 serial >> gpurun_out/qt.log 2>&1; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo tests $?
