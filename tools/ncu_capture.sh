#!/bin/bash
# ncu --set full captures of the top kernels of one c4 bench pass (run under gpurun).
set -x
OUT=${1:-gpurun_out}
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"proj_tc|energy_tc" -c 2 -o $OUT/prof_proj $CMD > $OUT/ncu_proj.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gram_kernel|split_kernel" -c 2 -o $OUT/prof_gram $CMD > $OUT/ncu_gram.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_gq|stats_kernel" -c 2 -o $OUT/prof_eig $CMD > $OUT/ncu_eig.log 2>&1
ls -la $OUT
