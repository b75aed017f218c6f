#!/bin/bash
# small-m split-K GEMM with more resident CTAs: GPU tests, c2 / c3 / c1-ish benches, c2 launch list
O=gpurun_out/g32; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
AVD_EIG_NOGRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:avd:: --csv --log-file $O/launches_c2.csv python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c2.log 2>&1
ls -la $O
