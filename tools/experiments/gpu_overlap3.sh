# Overlapped leaf groups as the default: full GPU suite, then c2 / c4 / c5-alt lines with parity
O=gpurun_out/ov3; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --workload c2-gf2-altsi-65536 --e2e-steps 20 > $O/bench_c2_altsi.log 2>&1
BMMGPU_ALT_OVERLAP=0 timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --no-check --e2e-steps 20 > $O/bench_c2_off.log 2>&1
timeout 900 python bench.py --workload c4-gf2-altsi-262144 --steps 3 --no-cpu-baseline --e2e-steps 2 > $O/bench_c4_altsi.log 2>&1
timeout 1500 python bench.py --workload c5-gf2-altooc-524288 --steps 1 --warmup 1 --check > $O/bench_c5_gf2_altooc.log 2>&1
tail -n 2 $O/pytest_gpu.log
for f in $O/bench_*.log; do echo $f; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline') or {}; e=d.get('e2e') or {}; print(d['value'], e.get('value'), r.get('frac'), r.get('sm_clock_effective_mhz'), (d.get('parity') or {}).get('ok'))"; done
