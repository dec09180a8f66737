#!/bin/bash
out=gpurun_out/ab_c2.log; : > $out
for ns in 8 16 24 32; do
  for gm in 4 3; do
    echo "== nseg $ns gmul $gm" >> $out
    SYLV_NSEG=$ns SYLV_G25MUL=$gm timeout 300 python tools/quick_time.py c2 20 serial 2>&1 | grep -E "pass1:|pass2:|ms/step" >> $out
  done
done
