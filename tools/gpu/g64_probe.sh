#!/bin/bash
# fp64 Rayleigh-Ritz product with 8 x 6 register tiles at c4: GPU suite, c4 benches, c4 launch list
O=gpurun_out/g64; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --variant massive --no-cpu-baseline > $O/bench_c4_massive.json 2> $O/bench_c4_massive.err
AVD_EIG_NOGRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:avd:: --csv --log-file $O/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c4.log 2>&1
ls -la $O
