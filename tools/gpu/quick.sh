#!/bin/bash
# quick GPU check: build, GPU tests, one bench line.  usage: bash tools/gpu/quick.sh TAG [pytest -k expr]
TAG=${1:-q}; K=${2:-}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/${TAG}_smoke.log
if [ -n "$K" ]; then timeout 900 python -m pytest tests -m gpu -x -q --timeout=150 -k "$K" > $OUT/${TAG}_pytest.log 2>&1
else timeout 900 python -m pytest tests -m gpu -x -q --timeout=150 > $OUT/${TAG}_pytest.log 2>&1; fi
echo "pytest rc=$?"; tail -15 $OUT/${TAG}_pytest.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench rc=$?"; cat $OUT/${TAG}_bench.json; tail -3 $OUT/${TAG}_bench.err
