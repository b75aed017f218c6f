#!/bin/bash
# launch list (ncu gpu__time_duration per kernel) of a short default bench run
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 ${BENCH_ARGS} > gpurun_out/b_ncu.log 2>&1
