#!/bin/bash
# Where the small-config step goes (c0, c2, c4): device step time with two streams vs serial,
# and the ncu launch list (durations only, serialised) of a few steps of each.
set -x
mkdir -p gpurun_out
out=gpurun_out/small_probe.log; : > $out
for c in c0 c2 c4; do
  echo "== $c two streams" >> $out
  timeout 300 python tools/quick_time.py $c 20 2>&1 | grep -E "ms/step|us/launch" >> $out
  echo "== $c serial" >> $out
  timeout 300 python tools/quick_time.py $c 20 serial 2>&1 | grep -E "ms/step|us/launch" >> $out
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/small_${c}_launches.csv \
    python tools/quick_time.py $c 5 > /dev/null 2>&1; echo "ncu $c $?" >> $out
done
