#!/bin/bash
# One GPU call: parity tests, a bench line, the launch list and ncu --set full captures.
# usage (under gpurun): bash tools/gpu/full_check.sh TAG "kernel_regex1" "kernel_regex2" ...
TAG=${1:-r01}; shift
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/${TAG}_smi.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q --timeout=600 > $OUT/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/${TAG}_pytest.log
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench rc=$?"; cat $OUT/${TAG}_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:avd:: -c 400 --csv --log-file $OUT/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo "launches rc=$?"
i=0
for RX in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s 2 -c 1 -o $OUT/${TAG}_prof_$i \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/${TAG}_ncu_$i.log 2>&1
  echo "ncu $RX rc=$?"; i=$((i+1))
done
ls -la $OUT
