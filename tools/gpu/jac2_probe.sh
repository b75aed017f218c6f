#!/bin/bash
# Jacobi stopping test relative to the larger column: GPU suite, c1 / c2 / c4 / c5 benches (sweeps per solve)
O=gpurun_out/jac2; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --variant massive --no-cpu-baseline > $O/bench_c4_massive.json 2> $O/bench_c4_massive.err
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err
ls -la $O
