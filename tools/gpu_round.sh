# round measurement: all GPU tests, bench (c3), ncu launch list of the same command
set -x
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider -o faulthandler_timeout=600 > gpurun_out/gputest.log 2>&1; echo tests $?
timeout 300 python tools/init_probe.py c3 > gpurun_out/init.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench $?
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ttt > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ttt > gpurun_out/ncu.log 2>&1; echo ncu $?
