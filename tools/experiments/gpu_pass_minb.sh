# Pass kernels' resident CTAs per SM: default (expand 2, compress 2) vs compress 3 (80 registers,
# 256 B spill) vs expand 3; c2 device, alternated on one box
O=gpurun_out/pm; mkdir -p $O
cp paper_1909_01554_b200/libbmmgpu.so $O/lib_default.so
run() {
  cp $2 paper_1909_01554_b200/libbmmgpu.so
  echo "== $1" >> $O/c2.txt
  timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --no-check --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],3), round(d['ms_per_step'],2), r.get('sm_clock_effective_mhz'))" >> $O/c2.txt 2>&1
}
for r in 1 2 3; do
  run default $O/lib_default.so
  run compress_minb3 build/variants/libbmmgpu_cminb3.so
  run expand_minb3 build/variants/libbmmgpu_eminb3.so
done
cp $O/lib_default.so paper_1909_01554_b200/libbmmgpu.so; rm -f $O/lib_default.so
cat $O/c2.txt
