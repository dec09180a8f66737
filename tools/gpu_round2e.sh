#!/bin/bash
# Round-2 final measurement after the sliding-ring CSR pass 1 (one gpurun call): bench lines for
# every BASELINE config and the paper workloads, the c3 launch list of the bench command (ncu,
# durations only), ncu --set full of the c4 hot kernels (both sequences) and the c3 passes + sketch.
set -x
tag=${1:-r2e}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${tag}_c3.json 2> gpurun_out/${tag}_c3.err; echo bench c3 $?
for c in c4 c2 c1 c0; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${tag}_$c.json 2> gpurun_out/${tag}_$c.err; done
for c in ex61_nu0.1 ex63_n125000; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/${tag}_$c.json 2> gpurun_out/${tag}_$c.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_c3_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ttt --no-near > gpurun_out/${tag}_ncu_launch.log 2>&1; echo ncu $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_c4_launches.csv python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ttt --no-near > gpurun_out/${tag}_ncu_launch4.log 2>&1; echo ncu $?
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "probe/" -k regex:"k_pass1_sell|k_pass2|k_sketch" -c 8 -o /tmp/${tag}_c4_full python tools/near_probe.py c4 5 1 > gpurun_out/${tag}_ncu_c4.log 2>&1; echo ncu4 $?
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "probe/" -k regex:"k_st3d|k_sketch_pull<" -c 3 -o /tmp/${tag}_c3_full python tools/near_probe.py c3 20 1 > gpurun_out/${tag}_ncu_c3.log 2>&1; echo ncu3 $?
for c in c3 c4; do
  ncu -i /tmp/${tag}_${c}_full.ncu-rep --page raw --csv > gpurun_out/${tag}_${c}_full_raw.csv 2>/dev/null
done
du -sh gpurun_out
