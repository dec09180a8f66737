timeout 300 python tools/e2e_probe.py > gpurun_out/e2e.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider -o faulthandler_timeout=600 > gpurun_out/gputest.log 2>&1; echo tests $?
