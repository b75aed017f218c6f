#!/bin/bash
# round-2 evidence set: bench lines (c4 default with the oracle baseline, c4 massive, c2, c3, c5,
# the reference arm), the launch list (host-loop eigensolver so ncu sees every kernel), and
# ncu --set full of the top kernels at c4.  Run under gpurun from the repo root.
mkdir -p gpurun_out/r2
O=gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --variant massive --no-cpu-baseline > $O/bench_c4_massive.json 2> $O/bench_c4_massive.err
timeout 600 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --impl reference > $O/bench_c4_reference.json 2> $O/bench_c4_reference.err
AVD_EIG_NOGRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/b_ncu.log 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
i=0
for RX in "gram2_kernel" "pass1_kernel" "proj_i8_kernel" "energy_tc_kernel" "sample_kernel"; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$RX" -c 1 -o $O/prof_$i $CMD > $O/ncu_$i.log 2>&1
  i=$((i+1))
done
ls -la $O
