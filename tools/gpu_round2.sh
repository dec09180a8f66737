#!/bin/bash
# Round-2 measurement (one gpurun call): bench lines for every BASELINE config and the paper
# workloads, the c3 launch list of the bench command (ncu, durations only), and ncu --set full
# captures of the hot kernels (c3 passes + sketch, c4 SELL pass 1, c2 passes).
set -x
tag=${1:-r2}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${tag}_c3.json 2> gpurun_out/${tag}_c3.err; echo bench c3 $?
for c in c2 c4 c1 c0; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${tag}_$c.json 2> gpurun_out/${tag}_$c.err; done
for c in ex61_nu0.1 ex63_n125000; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/${tag}_$c.json 2> gpurun_out/${tag}_$c.err; done
SYLV_TRACE_PROJ=1 timeout 600 python tools/ttt.py c2 > gpurun_out/${tag}_ttt_c2.log 2>&1
SYLV_TRACE_PROJ=1 timeout 600 python tools/ttt.py c3 > gpurun_out/${tag}_ttt_c3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_c3_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ttt --no-near > gpurun_out/${tag}_ncu_launch.log 2>&1; echo ncu $?
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "probe/" -k regex:"k_st3d|k_sketch_pull<|k_qtw|k_qc_part|k_qc_mma" -c 6 -o /tmp/${tag}_c3_full python tools/near_probe.py c3 204 1 > gpurun_out/${tag}_ncu_c3.log 2>&1; echo ncu3 $?
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "probe/" -k regex:"k_pass1_sell|k_pass2|k_sketch" -c 4 -o /tmp/${tag}_c4_full python tools/near_probe.py c4 5 1 > gpurun_out/${tag}_ncu_c4.log 2>&1; echo ncu4 $?
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "probe/" -k regex:"k_st3d|k_sketch" -c 4 -o /tmp/${tag}_c2_full python tools/near_probe.py c2 20 1 > gpurun_out/${tag}_ncu_c2.log 2>&1; echo ncu2 $?
# the .ncu-rep files stay on the box (gpurun_out is capped at 64 MiB): raw metrics as CSV
for c in c3 c4 c2; do
  ncu -i /tmp/${tag}_${c}_full.ncu-rep --page raw --csv > gpurun_out/${tag}_${c}_full_raw.csv 2>/dev/null
  ncu -i /tmp/${tag}_${c}_full.ncu-rep --page details --csv > gpurun_out/${tag}_${c}_full_details.csv 2>/dev/null
done
du -sh gpurun_out
