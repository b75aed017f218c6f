#!/bin/bash
# round-2 closing evidence for the final build: smoke, GPU suite, c1 / c2 / c3 / c4 (+ oracle baseline) /
# c4 massive / c5 benches, c4 and c1 launch lists (host-loop eigensolver), ncu of the row sample
O=gpurun_out/r9; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --variant massive --no-cpu-baseline > $O/bench_c4_massive.json 2> $O/bench_c4_massive.err
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err
AVD_EIG_NOGRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:avd:: --csv --log-file $O/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_c4.log 2>&1
AVD_EIG_NOGRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:avd:: --csv --log-file $O/launches_c1.csv python bench.py --config c1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:sample_kernel -c 1 -o $O/prof_sample python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_sample.log 2>&1
ls -la $O
