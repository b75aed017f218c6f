#!/bin/bash
# graph-conditional probe, massive-activation bench line, launch list of the default bench
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/gcp tools/graph_cond_probe.cu && timeout 60 /tmp/gcp > gpurun_out/gcp.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --variant massive > gpurun_out/bench_massive.json 2> gpurun_out/bench_massive.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_ncu.log 2>&1
