#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-ay}
AVD_AV_CFG=2 timeout 600 python -m pytest tests/test_gpu_averis.py -x -q > $OUT/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/${TAG}_pytest.log
for C in 0 2; do for D in 0 1; do
  AVD_AV_CFG=$C AVD_AV_DBG=$D timeout 300 python bench.py --config averis --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/${TAG}_c${C}_d$D.json 2>&1
done; done
