# after the non-blocking free-memory estimate: first-call cost (fresh processes), c4 alt-si and c5 alt out-of-core lines
mkdir -p gpurun_out/am
O=gpurun_out/am
: > $O/first_call.txt
for mode in none plain reserve; do timeout 300 python microbench/first_call.py 65536 $mode >> $O/first_call.txt 2>&1; done
cat $O/first_call.txt
timeout 900 python bench.py --workload c4-gf2-altsi-262144 --steps 3 --no-cpu-baseline --e2e-steps 3 > $O/c4.log 2>&1
timeout 1500 python bench.py --workload c5-gf2-altooc-524288 --steps 1 --warmup 1 > $O/c5.log 2>&1
for f in $O/c4.log $O/c5.log; do python -c "
import json
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; e=d['e2e']; print('$f', round(d['value'],3), round(d['ms_per_step'],1), 'e2e', round(e['value'],3), e.get('samples_ms'), r.get('frac'), r.get('sm_clock_effective_mhz'), r.get('frac_per_clock'), (d.get('parity') or {}).get('ok'))
"; done
free -g | head -2
