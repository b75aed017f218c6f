#!/bin/bash
# f3 check: parity tests, the averis bench line, the launch list and ncu of the GeMM / quantiser
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-av}
timeout 600 python -m pytest tests/test_gpu_averis.py -x -q > $OUT/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/${TAG}_pytest.log
timeout 600 python bench.py --config averis --steps 20 --warmup 3 > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench rc=$?" >> $OUT/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:av_ -c 40 --csv --log-file $OUT/${TAG}_launches.csv \
  python bench.py --config averis --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "launches rc=$?"
for RX in av_gemm_kernel av_quant_rows_kernel av_colstats_kernel; do C=1; [ $RX = av_quant_rows_kernel ] && C=2
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$RX -s 4 -c $C -o $OUT/${TAG}_prof_$RX \
    python bench.py --config averis --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/${TAG}_ncu_$RX.log 2>&1; echo "ncu $RX rc=$?"
done
