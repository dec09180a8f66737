for c in c0 c2 c3; do timeout 300 python tools/ttt.py $c >> gpurun_out/ttt.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "solve" -o faulthandler_timeout=300 > gpurun_out/gputest.log 2>&1; echo tests $?
