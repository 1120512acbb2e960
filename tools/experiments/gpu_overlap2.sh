# Overlapped leaf groups, end to end (streamed children at n/2 have 49 leaves per group):
# group size threshold and the leaves' stream priority, alternated on one box.
O=gpurun_out/ov2; mkdir -p $O
run() {  # label, env...
  echo "== $1" >> $O/c2.txt; shift
  env "$@" timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --no-check --e2e-steps 20 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],3), round(d['ms_per_step'],2), round(d['e2e']['value'],3), r.get('sm_clock_effective_mhz'))" >> $O/c2.txt 2>&1
}
for r in 1 2; do
  run off BMMGPU_ALT_OVERLAP=0
  run min49_prio1 BMMGPU_ALT_OVERLAP=1 BMMGPU_ALT_OVERLAP_MIN=49
  run min49_prio0 BMMGPU_ALT_OVERLAP=1 BMMGPU_ALT_OVERLAP_MIN=49 BMMGPU_ALT_OVERLAP_PRIO=0
  run min343 BMMGPU_ALT_OVERLAP=1 BMMGPU_ALT_OVERLAP_MIN=343
  run min49_ov2 BMMGPU_ALT_OVERLAP=2 BMMGPU_ALT_OVERLAP_MIN=49
done
BMMGPU_ALT_TRACE=1 BMMGPU_ALT_OVERLAP=0 timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --no-check --e2e-steps 3 --steps 2 > $O/trace_off.log 2>&1
BMMGPU_ALT_TRACE=1 BMMGPU_ALT_OVERLAP=1 timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --no-check --e2e-steps 3 --steps 2 > $O/trace_on.log 2>&1
cat $O/c2.txt
