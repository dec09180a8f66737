timeout 900 python -m pytest tests/test_gpu_sketch_pull.py tests/test_gpu_sharded.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -o faulthandler_timeout=300 -k "pull or full_config or sharded" > gpurun_out/pt.log 2>&1; echo tests $? >> gpurun_out/pt.log
for c in c4 c3 c2 c1; do timeout 300 python tools/quick_time.py $c 20 2>&1 | grep -E "ms/step" >> gpurun_out/fold.log; done
