set -x
for a in "34 3" "64 3" "26 4"; do timeout 120 python tools/small_tma.py $a 2>&1 | tail -1; done > gpurun_out/dbg.log 2>&1
timeout 600 python tools/quick_time.py c3 10 serial > gpurun_out/qt.log 2>&1; echo qt $?
timeout 900 python -m pytest tests -m gpu -x -q -k "tma" > gpurun_out/gputest.log 2>&1; echo tests $?
timeout 300 python tools/quick_time.py c3 10 >> gpurun_out/qt.log 2>&1
timeout 300 python tools/quick_time.py c3 10 serial > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sketch_cols|k_st3d_r8" -s 2 -c 4 -o gpurun_out/prof_r1b python tools/quick_time.py c3 10 serial > gpurun_out/ncu.log 2>&1; echo ncu $?
