#!/bin/bash
# K5/K8 check: parity tests, bench, ncu of both kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err
bash tools/gpu/ncu_one.sh k5 "proj_i8_kernel"; bash tools/gpu/ncu_one.sh k8 "energy_i8_kernel"
