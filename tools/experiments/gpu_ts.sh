# A-in-TMEM K2 mode (kTs) for long-K launches: parity tests, then the c3 bench against the SS-only build
mkdir -p gpurun_out/ts
timeout 900 python -m pytest tests/test_cubic_gpu.py tests/test_dropin.py -m gpu -x -q -s -k "tmem or kernel64 or wave or long or large or accumulate or random or out_of_core or concurrent or fp32" > gpurun_out/ts/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ts/pytest.log
tail -3 gpurun_out/ts/pytest.log
grep 'kernel64:' gpurun_out/ts/pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ts/bench_c3_ts.log 2>&1
BMMGPU_TS_MIN_STAGES=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ts/bench_c3_ss.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ts/bench_c3_ts2.log 2>&1
for f in gpurun_out/ts/bench_*.log; do echo $f; python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d.get('e2e',{}) and d['e2e']['value'], d['roofline']['kernel_ms'], d['clocks'], d.get('parity',{}).get('ok'))
"; done
