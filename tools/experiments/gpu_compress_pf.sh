# Group compresses beside the leaves with a capped grid and L2 bulk prefetch (BMMGPU_COMPRESS_PF=blocks)
O=gpurun_out/pf; mkdir -p $O
BMMGPU_COMPRESS_PF=296 timeout 600 python -m pytest tests/test_alt_gpu.py -m gpu -x -q > $O/pytest_alt_pf.log 2>&1; echo "rc=$?" >> $O/pytest_alt_pf.log
run() {
  echo "== $1" >> $O/c2.txt; shift
  env "$@" timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --no-check --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],3), round(d['ms_per_step'],2), r.get('sm_clock_effective_mhz'))" >> $O/c2.txt 2>&1
}
for r in 1 2; do
  run base
  run pf296 BMMGPU_COMPRESS_PF=296
  run pf592 BMMGPU_COMPRESS_PF=592
  run pf296_o1_ov1 BMMGPU_COMPRESS_PF=296 BMMGPU_ALT_OVERLAP_ORDER=1
  run pf296_o1_ov2 BMMGPU_COMPRESS_PF=296 BMMGPU_ALT_OVERLAP_ORDER=1 BMMGPU_ALT_OVERLAP=2
done
for v in "BMMGPU_COMPRESS_PF=296" "BMMGPU_COMPRESS_PF=296 BMMGPU_ALT_OVERLAP_ORDER=1"; do
  env $v BMMGPU_GROUP_TRACE=1 timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --no-check --no-e2e --steps 3 --warmup 3 2>&1 | grep groups | tail -1 >> $O/trace.txt
done
tail -2 $O/pytest_alt_pf.log; cat $O/c2.txt $O/trace.txt
