# A-in-TMEM (kTs) vs both operands in shared memory for long-K launches: TS parity test, then the c3
# device bench alternated 3 x each (BMMGPU_TS_MIN_STAGES=0 disables kTs), with the K2 effective clock
mkdir -p gpurun_out/ts
timeout 600 python -m pytest tests/test_cubic_gpu.py -m gpu -x -q -k "tmem" > gpurun_out/ts/pytest2.log 2>&1; echo "rc=$?" >> gpurun_out/ts/pytest2.log
tail -2 gpurun_out/ts/pytest2.log
: > gpurun_out/ts/ab.txt
for i in 1 2 3; do
  for mode in 128 0; do
    BMMGPU_TS_MIN_STAGES=$mode timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-check --steps 5 > gpurun_out/ts/ab_$mode.log 2>&1
    python -c "
import json
for l in open('gpurun_out/ts/ab_$mode.log'):
    if l.startswith('{'):
        d=json.loads(l); print('ts_min=$mode', round(d['value'],4), round(d['roofline']['kernel_ms'],2), d['roofline'].get('sm_clock_effective_mhz'), d['roofline'].get('frac_per_clock'), d['clocks']['sm_mhz'])
" >> gpurun_out/ts/ab.txt
  done
done
cat gpurun_out/ts/ab.txt
