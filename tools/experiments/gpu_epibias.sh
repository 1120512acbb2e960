# accumulator bias written by the epilogue (default) vs the per-tile bias MMA (biasmma variant), and the
# 16-column accumulator overlap (ovl16 variant): GPU parity suite on the default and ovl16 builds, then
# leaf batches and the c2 device bench alternated
mkdir -p gpurun_out/eb
O=gpurun_out/eb
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
cp paper_1909_01554_b200/libbmmgpu.so /tmp/libbmmgpu.new.so
cp build/variants/libbmmgpu_ovl16.so paper_1909_01554_b200/libbmmgpu.so
timeout 900 python -m pytest tests/test_cubic_gpu.py tests/test_alt_gpu.py -m gpu -x -q > $O/pytest_ovl16.log 2>&1; echo "rc=$?" >> $O/pytest_ovl16.log
tail -2 $O/pytest_ovl16.log
: > $O/ab.txt
for i in 1 2; do
  for v in new biasmma ovl16; do
    if [ $v = new ]; then cp /tmp/libbmmgpu.new.so paper_1909_01554_b200/libbmmgpu.so; else cp build/variants/libbmmgpu_$v.so paper_1909_01554_b200/libbmmgpu.so; fi
    echo "== $v" >> $O/ab.txt
    timeout 300 python microbench/time_leaf.py 4096,2048 >> $O/ab.txt 2>&1
    timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --no-e2e --no-check --steps 5 > $O/c2_$v.log 2>&1
    python -c "
import json
for l in open('$O/c2_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print('c2', round(d['value'],4), round(r['kernel_ms'],3), r.get('sm_clock_effective_mhz'), r.get('frac_per_clock'))
" >> $O/ab.txt
  done
done
cp /tmp/libbmmgpu.new.so paper_1909_01554_b200/libbmmgpu.so
cat $O/ab.txt
