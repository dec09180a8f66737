# round measurement: tests, bench (c3), launch list
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo tests $?
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench $?
for c in c2 c1; do timeout 600 python tools/ttt.py $c >> gpurun_out/ttt.log 2>&1; done
