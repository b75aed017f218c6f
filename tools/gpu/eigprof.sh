#!/bin/bash
# eigensolver profile: host-driven mode (every kernel visible to ncu): launch list + ncu --set full
# of the fp32 GEMM and the Rayleigh-Ritz Jacobi; then the graph-mode bench
mkdir -p gpurun_out
export AVD_EIG_NOGRAPH=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu.log 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_kernel<float" -c 1 -o gpurun_out/prof_gemm32 $CMD > gpurun_out/ncu_g.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"atb_fused_kernel<2" -c 1 -o gpurun_out/prof_atb2 $CMD > gpurun_out/ncu_a.log 2>&1
unset AVD_EIG_NOGRAPH
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err
