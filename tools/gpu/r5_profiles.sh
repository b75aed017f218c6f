#!/bin/bash
# round-2 (final session) evidence set: bench lines (c4 default with the oracle baseline, c4 massive,
# c2, c3, c5, averis, reference arms), launch lists (host-loop eigensolver so ncu sees every kernel;
# averis), ncu --set full of the top kernels.  Run under gpurun from the repo root.
O=gpurun_out/r5; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --config averis > $O/bench_averis.json 2> $O/bench_averis.err
timeout 600 python bench.py --config averis --variant bf16 --no-cpu-baseline > $O/bench_averis_bf16.json 2> $O/bench_averis_bf16.err
timeout 600 python bench.py --variant gramfree --no-cpu-baseline > $O/bench_c4_gramfree.json 2> $O/bench_c4_gramfree.err
timeout 600 python bench.py --variant massive --no-cpu-baseline > $O/bench_c4_massive.json 2> $O/bench_c4_massive.err
timeout 600 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --config c5 --variant gramfree --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c5_gramfree.json 2> $O/bench_c5_gramfree.err
timeout 600 python bench.py --impl reference > $O/bench_c4_reference.json 2> $O/bench_c4_reference.err
timeout 600 python bench.py --impl reference --config averis --steps 3 > $O/bench_averis_reference.json 2> $O/bench_averis_reference.err
AVD_EIG_NOGRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:avd:: --csv --log-file $O/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/b_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:avd:: --csv --log-file $O/launches_c4_gramfree.csv python bench.py --variant gramfree --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:av_ --csv --log-file $O/launches_averis.csv python bench.py --config averis --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
i=0
for RX in "gram2_kernel" "pass1_kernel" "proj_i8_kernel" "energy_i8_kernel" "gf_xq_kernel" "gf_xtp_kernel"; do
  EXTRA=""; case $RX in gf_*) EXTRA="--variant gramfree";; esac
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$RX" -c 1 -o $O/prof_$i $CMD $EXTRA > $O/ncu_$i.log 2>&1
  i=$((i+1))
done
for RX in av_gemm_kernel av_quant_rows_kernel; do C=1; [ $RX = av_quant_rows_kernel ] && C=2
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$RX -s 4 -c $C -o $O/prof_$RX \
    python bench.py --config averis --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_$RX.log 2>&1
done
ls -la $O
