#!/bin/bash
# half-warp Jacobi check: GPU tests, c4 / c2 benches, launch lists of c4 and c2 (host-loop eig)
O=gpurun_out/jac; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
AVD_EIG_NOGRAPH=1 timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $O/bench_c2_nograph.json 2> $O/bench_c2_nograph.err
AVD_EIG_NOGRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:avd:: --csv --log-file $O/launches_c2.csv python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c2.log 2>&1
AVD_EIG_NOGRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:avd:: --csv --log-file $O/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c4.log 2>&1
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err
ls -la $O
