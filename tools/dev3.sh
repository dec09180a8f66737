#!/bin/bash
# development call: register / threads variants of the ring SELL pass 1 (c4)
out=gpurun_out/dev3.log; : > $out
for v in base ne8 t512ne8 t512ne16; do
  if [ $v = base ]; then unset SYLV_LIB_PATH; else export SYLV_LIB_PATH=$PWD/ab_libs/libsylvsketch_$v.so; fi
  echo "== c4 $v serial" >> $out
  timeout 200 python tools/quick_time.py c4 20 serial 2>&1 | grep -E "pass1:|sketch:|ms/step" >> $out
done
unset SYLV_LIB_PATH
echo "== c4 base two-stream" >> $out
timeout 200 python tools/quick_time.py c4 40 2>&1 | grep -E "ms/step" >> $out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_pass1_sell_ring|k_sketch_pull" -s 6 -c 4 -o /tmp/dev3_c4 python tools/quick_time.py c4 6 serial > gpurun_out/dev3_ncu.log 2>&1
ncu -i /tmp/dev3_c4.ncu-rep --page raw --csv > gpurun_out/dev3_c4_raw.csv 2>/dev/null
ncu -i /tmp/dev3_c4.ncu-rep --page source --csv -k regex:k_pass1_sell_ring > gpurun_out/dev3_c4_source.csv 2>/dev/null
cat $out
