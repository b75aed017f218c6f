#!/bin/bash
# ncu --set full of ONE kernel (regex on the demangled name) of a short bench run: ncu_one.sh NAME REGEX [env...]
mkdir -p gpurun_out
NAME=$1; RX=$2
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$RX" -c 1 -o gpurun_out/prof_$NAME $CMD > gpurun_out/ncu_$NAME.log 2>&1
tail -3 gpurun_out/ncu_$NAME.log
