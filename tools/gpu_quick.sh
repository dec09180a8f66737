timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -o faulthandler_timeout=600 > gpurun_out/gputest.log 2>&1; echo tests $? >> gpurun_out/gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke $? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench $? >> gpurun_out/smoke.log
