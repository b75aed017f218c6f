timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout=300 -k "c1 or ragged or planted" 2>&1 | tail -2
for S in 0 5 7 11 16 22 32; do
  if [ $S = 0 ]; then unset AVD_GRAM_SPLIT; else export AVD_GRAM_SPLIT=$S; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('S=$S', round(d['ms_per_step'],3), 'gram_launch', round(d['roofline']['launch_ms'],3), 'stage', round(d['stage_ms']['gram'],3))"
done
export AVD_GRAM_SPLIT=16
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:gram_kernel -c 1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | grep -E "dram__|gpu__time" 
unset AVD_GRAM_SPLIT
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:gram_kernel -c 1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | grep -E "dram__|gpu__time" 
