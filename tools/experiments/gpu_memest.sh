# non-blocking free-memory estimate (device_free_bytes): GPU suite, c2 per-step host enqueue, c2 / c3 bench with e2e samples
mkdir -p gpurun_out/me
O=gpurun_out/me
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
timeout 200 python microbench/c2_steps.py 65536 10 > $O/steps.txt 2>&1
timeout 200 python microbench/c2_steps.py 65536 10 >> $O/steps.txt 2>&1
cat $O/steps.txt | cut -c1-400
timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --e2e-steps 20 > $O/c2.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > $O/c3.log 2>&1
for f in $O/c2.log $O/c3.log; do python -c "
import json
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; e=d['e2e']; print('$f', round(d['value'],3), round(d['ms_per_step'],2), 'e2e', round(e['value'],3), e.get('samples_ms'), r.get('sm_clock_effective_mhz'), r.get('frac_per_clock'), d['parity']['ok'])
"; done
