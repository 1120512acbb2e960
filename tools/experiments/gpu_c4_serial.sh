# c4 (n=262144): depth-first levels 1 vs 2 (BMMGPU_ALT_SERIAL) with the overlapped leaf groups' smaller footprint
O=gpurun_out/c4s; mkdir -p $O
run() {
  echo "== $1" >> $O/c4.txt; shift
  env "$@" timeout 900 python bench.py --workload c4-gf2-altsi-262144 --steps 2 --no-cpu-baseline --no-check --e2e-steps 1 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; e=d.get('e2e') or {}; print(round(d['value'],3), round(d['ms_per_step'],1), e.get('value') and round(e['value'],3), r.get('sm_clock_effective_mhz'))" >> $O/c4.txt 2>&1
}
for r in 1 2; do
  run serial_default
  run serial1 BMMGPU_ALT_SERIAL=1
done
cat $O/c4.txt
