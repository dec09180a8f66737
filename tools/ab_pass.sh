#!/bin/bash
# A/B of pass-kernel variants (build_ab/*.so via SYLV_LIB_PATH) on c3 and c2, serial attribution
out=gpurun_out/ab_pass.log; : > $out
for v in base "$@"; do
  if [ $v = base ]; then unset SYLV_LIB_PATH; else export SYLV_LIB_PATH=$PWD/build_ab/libsylvsketch_$v.so; fi
  for c in c3 c2; do
    echo "== $v $c" >> $out
    timeout 300 python tools/quick_time.py $c 20 serial 2>&1 | grep -E "pass1|pass2|ms/step" >> $out
  done
done
unset SYLV_LIB_PATH
