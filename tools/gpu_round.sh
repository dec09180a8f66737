# round measurement, two gpurun calls (one ncu each):
#   bash tools/gpu_round.sh A : all GPU tests, bench (c3 + others), launch list of the bench command
#   bash tools/gpu_round.sh B : ncu --set full of the steady-state hot kernels (c3)
set -x
if [ "$1" = "A" ]; then
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider -o faulthandler_timeout=600 > gpurun_out/gputest.log 2>&1; echo tests $?
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench $?
for c in c2 c4 c1 c0; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ttt > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ttt > gpurun_out/ncu.log 2>&1; echo ncu $?
else
timeout 300 python tools/quick_time.py c3 4 serial > gpurun_out/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_st3d|k_sketch_pull" -s 20 -c 3 -o gpurun_out/prof_c3 python tools/quick_time.py c3 4 serial > gpurun_out/ncu2.log 2>&1; echo ncufull $?
fi
