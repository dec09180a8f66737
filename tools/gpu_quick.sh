for a in "32 8 3 2 6 notma" "32 8 2 2 6 tma" "34 8 3 3 6 tma"; do echo "== $a"; timeout 60 python tools/sharded_probe.py $a 2>&1 | grep "rank 0 step"; done > gpurun_out/probe2.log 2>&1
for i in 1 2; do timeout 600 python -m pytest tests/test_gpu_sharded.py -q -p no:cacheprovider >> gpurun_out/gputest.log 2>&1; echo tests $?; done
