# out-of-core fast product through device-generated sub-instances: tests, then the c5 alt line (sub-instances vs tiles)
mkdir -p gpurun_out/si
O=gpurun_out/si
timeout 900 python -m pytest tests/test_alt_gpu.py tests/test_multidevice.py tests/test_dropin.py -m gpu -q -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
tail -3 $O/pytest.log
timeout 1500 python bench.py --workload c5-gf2-altooc-524288 --steps 1 --warmup 1 > $O/c5_subinst.log 2>&1
BMMGPU_ALT_OOC=tiles timeout 1500 python bench.py --workload c5-gf2-altooc-524288 --steps 1 --warmup 1 --no-check > $O/c5_tiles.log 2>&1
for f in $O/c5_*.log; do python -c "
import json
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print('$f', round(d['value'],3), round(d['ms_per_step'],1), r['kernel_ms'], r['frac'], d['e2e']['h2d_bytes_per_step']/1e9, d['e2e']['d2h_bytes_per_step']/1e9, (d.get('parity') or {}).get('ok'), d['config']['driver'][:60])
"; done
tail -n 3 $O/c5_subinst.log | cut -c1-300
