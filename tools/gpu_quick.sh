timeout 900 python tools/proj_probe2.py > gpurun_out/proj2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "device_projected or with_device or full_solve" > gpurun_out/gputest.log 2>&1; echo tests $?
for c in c2 c3; do timeout 600 python tools/ttt.py $c >> gpurun_out/ttt.log 2>&1; done
