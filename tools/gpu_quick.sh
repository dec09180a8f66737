for c in c0 c4 c2; do timeout 900 python tools/ttt.py $c >> gpurun_out/ttt.log 2>&1; done
nproc >> gpurun_out/ttt.log; lscpu | grep "Model name" >> gpurun_out/ttt.log
