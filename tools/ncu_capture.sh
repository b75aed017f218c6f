#!/bin/bash
# ncu --set full captures of selected kernels of one c4 bench pass (run under gpurun).
# usage: tools/ncu_capture.sh OUT "regex1" "regex2" ...
OUT=${1:-gpurun_out}; shift
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
i=0
for RX in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" -c 1 -o $OUT/prof_$i $CMD > $OUT/ncu_$i.log 2>&1
  i=$((i+1))
done
ls -la $OUT
