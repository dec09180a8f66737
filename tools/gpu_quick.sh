timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -o faulthandler_timeout=300 -k "solve" > gpurun_out/pt.log 2>&1; echo tests $? >> gpurun_out/pt.log
for c in c1 c3 c2; do timeout 900 python tools/ttt.py $c > gpurun_out/ttt_$c.log 2>&1; done
