# sub-instance driver (4 host Q slots): tests, then the c5 alt line with the host-side trace
mkdir -p gpurun_out/si3
O=gpurun_out/si3
timeout 900 python -m pytest tests/test_alt_gpu.py -m gpu -q -x -k "out_of_core" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
tail -2 $O/pytest.log
BMMGPU_SUBINST_TRACE=1 timeout 1500 python bench.py --workload c5-gf2-altooc-524288 --steps 2 --warmup 1 > $O/c5.log 2>&1
grep subinst $O/c5.log
python -c "
import json
for l in open('$O/c5.log'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(round(d['value'],3), round(d['ms_per_step'],1), r['kernel_ms'], r['frac'], d['e2e']['h2d_bytes_per_step']/1e9, (d.get('parity') or {}).get('ok'))
"
