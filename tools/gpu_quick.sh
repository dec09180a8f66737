set -x
timeout 120 python tools/proj_probe.py > gpurun_out/proj.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "device_projected or with_device" > gpurun_out/gputest.log 2>&1; echo tests $?
for c in c2 c4; do timeout 300 python tools/ttt.py $c >> gpurun_out/ttt.log 2>&1; done
timeout 900 python tools/ttt.py c3 >> gpurun_out/ttt.log 2>&1; echo c3 $?
