#!/bin/bash
out=gpurun_out/ab_sched.log; : > $out
for c in c2 c4 c1; do
  for v in phase overlap; do
    echo "== $c $v" >> $out
    SYLV_SCHED=$v timeout 300 python tools/quick_time.py $c 40 2>&1 | grep -E "ms/step" >> $out
  done
done
