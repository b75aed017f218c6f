#!/bin/bash
# closing check of the committed final build: smoke, GPU suite, the default bench line (c4 with the
# oracle baseline) and the reference arm
O=gpurun_out/r10; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --config averis --no-cpu-baseline > $O/bench_averis.json 2> $O/bench_averis.err
timeout 600 python bench.py --impl reference > $O/bench_c4_reference.json 2> $O/bench_c4_reference.err
ls -la $O
