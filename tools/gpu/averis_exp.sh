#!/bin/bash
# f3 GeMM timing experiments (AVD_AV_DBG knobs) + parity
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-ax}
timeout 600 python -m pytest tests/test_gpu_averis.py -x -q > $OUT/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/${TAG}_pytest.log
for D in 0 1 2 4 6; do
  AVD_AV_DBG=$D timeout 300 python bench.py --config averis --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/${TAG}_dbg$D.json 2>&1
done
