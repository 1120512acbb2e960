# Expand pass compiled for 2 resident CTAs per SM (128 registers, small spill) vs 1 (140 registers):
# with 2 the side SMs beside the leaf launches hold twice the loads in flight, so the expand of
# group g + 2 may fit beside the leaves (order 1, 2-3 reserved pairs).  c2 device, alternated.
O=gpurun_out/em; mkdir -p $O
cp paper_1909_01554_b200/libbmmgpu.so $O/lib_minb2.so
BMMGPU_ALT_OVERLAP_ORDER=1 BMMGPU_ALT_OVERLAP=2 timeout 600 python -m pytest tests/test_alt_gpu.py -m gpu -x -q > $O/pytest_alt.log 2>&1; echo "rc=$?" >> $O/pytest_alt.log
run() {
  echo "== $1" >> $O/c2.txt; shift
  env "$@" timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --no-check --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],3), round(d['ms_per_step'],2), r.get('sm_clock_effective_mhz'))" >> $O/c2.txt 2>&1
}
for r in 1 2; do
  cp build/variants/libbmmgpu_minb1.so paper_1909_01554_b200/libbmmgpu.so
  run minb1_o0_ov1
  cp $O/lib_minb2.so paper_1909_01554_b200/libbmmgpu.so
  run minb2_o0_ov1
  run minb2_o1_ov2 BMMGPU_ALT_OVERLAP_ORDER=1 BMMGPU_ALT_OVERLAP=2
  run minb2_o1_ov3 BMMGPU_ALT_OVERLAP_ORDER=1 BMMGPU_ALT_OVERLAP=3
  run minb2_o0_ov2 BMMGPU_ALT_OVERLAP=2
done
for v in "BMMGPU_ALT_OVERLAP_ORDER=1 BMMGPU_ALT_OVERLAP=2" "BMMGPU_ALT_OVERLAP_ORDER=1 BMMGPU_ALT_OVERLAP=3"; do
  env $v BMMGPU_GROUP_TRACE=1 timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --no-check --no-e2e --steps 3 --warmup 3 2>&1 | grep groups | tail -1 >> $O/trace.txt
done
tail -2 $O/pytest_alt.log; cat $O/c2.txt $O/trace.txt
