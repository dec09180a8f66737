#!/bin/bash
# One bench line per BASELINE config (c3 is the default workload) into gpurun_out/<tag>_<cfg>.json
tag=${1:-r2}
shift
for c in ${@:-c3 c2 c4 c1 c0}; do
  python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/${tag}_${c}.json 2> gpurun_out/${tag}_${c}.err
done
