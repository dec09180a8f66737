#!/bin/bash
# development call: schedule A/B on the small configs, c2 serial split and launch list
out=gpurun_out/dev1.log; : > $out
for c in c2 c1 c0; do
  for v in phase overlap; do
    echo "== $c $v" >> $out
    SYLV_SCHED=$v timeout 300 python tools/quick_time.py $c 40 2>&1 | grep -E "ms/step" >> $out
  done
done
echo "== c2 serial" >> $out
timeout 300 python tools/quick_time.py c2 40 serial 2>&1 | grep -E "ms/step|us/launch" >> $out
echo "== c3" >> $out
timeout 300 python tools/quick_time.py c3 20 2>&1 | grep -E "ms/step" >> $out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dev1_c2_launches.csv python tools/quick_time.py c2 4 > gpurun_out/dev1_ncu.log 2>&1
python tools/ncu_summary.py launches gpurun_out/dev1_c2_launches.csv gpurun_out/dev1_c2_summary.json >/dev/null 2>&1
cat $out
