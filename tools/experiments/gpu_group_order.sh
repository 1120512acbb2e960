# Pass-stream order of the overlapped leaf groups: 0 = compress g then expand g+2 (2 Q slots),
# 1 = expand g+2 then compress g (3 Q slots); reserved CTA pairs swept; c2 device, alternated
O=gpurun_out/go; mkdir -p $O
BMMGPU_ALT_OVERLAP_ORDER=1 timeout 600 python -m pytest tests/test_alt_gpu.py -m gpu -x -q > $O/pytest_alt_order1.log 2>&1; echo "rc=$?" >> $O/pytest_alt_order1.log
run() {
  echo "== $1" >> $O/c2.txt; shift
  env "$@" timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --no-check --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],3), round(d['ms_per_step'],2), r.get('sm_clock_effective_mhz'))" >> $O/c2.txt 2>&1
}
for r in 1 2; do
  run o0_ov1 BMMGPU_ALT_OVERLAP_ORDER=0 BMMGPU_ALT_OVERLAP=1
  run o1_ov2 BMMGPU_ALT_OVERLAP_ORDER=1 BMMGPU_ALT_OVERLAP=2
  run o1_ov3 BMMGPU_ALT_OVERLAP_ORDER=1 BMMGPU_ALT_OVERLAP=3
  run o1_ov4 BMMGPU_ALT_OVERLAP_ORDER=1 BMMGPU_ALT_OVERLAP=4
  run o1_ov6 BMMGPU_ALT_OVERLAP_ORDER=1 BMMGPU_ALT_OVERLAP=6
  run o0_ov3 BMMGPU_ALT_OVERLAP_ORDER=0 BMMGPU_ALT_OVERLAP=3
done
for ov in 3 4; do
  BMMGPU_GROUP_TRACE=1 BMMGPU_ALT_OVERLAP_ORDER=1 BMMGPU_ALT_OVERLAP=$ov timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --no-check --no-e2e --steps 3 --warmup 3 > $O/trace_o1_ov$ov.log 2>&1
done
tail -2 $O/pytest_alt_order1.log; cat $O/c2.txt; grep groups $O/trace_o1_ov3.log | tail -1; grep groups $O/trace_o1_ov4.log | tail -1
