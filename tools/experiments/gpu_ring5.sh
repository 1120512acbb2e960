# K2 with a 5-stage operand ring (bias written by the epilogue frees the 16 KB constant region) vs the
# default (4 stages, bias MMA) and the 4-stage epilogue-bias build: parity on the eb5 build, then leaf
# batches, c2 and c3 device lines alternated
mkdir -p gpurun_out/r5
O=gpurun_out/r5
cp paper_1909_01554_b200/libbmmgpu.so /tmp/def.so
cp build/variants/libbmmgpu_eb5.so paper_1909_01554_b200/libbmmgpu.so
timeout 900 python -m pytest tests/test_cubic_gpu.py tests/test_alt_gpu.py -m gpu -q -x > $O/pytest_eb5.log 2>&1; echo rc=$? >> $O/pytest_eb5.log
tail -2 $O/pytest_eb5.log
: > $O/ab.txt
for i in 1 2; do
  for v in def eb5 eb4; do
    if [ $v = def ]; then cp /tmp/def.so paper_1909_01554_b200/libbmmgpu.so; else cp build/variants/libbmmgpu_$v.so paper_1909_01554_b200/libbmmgpu.so; fi
    echo "== $v" >> $O/ab.txt
    timeout 300 python microbench/time_leaf.py 4096 >> $O/ab.txt 2>&1
    timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --no-e2e --no-check --steps 8 > $O/c2_$v.log 2>&1
    timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-check --steps 4 > $O/c3_$v.log 2>&1
    for w in c2 c3; do python -c "
import json
for l in open('$O/${w}_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print('$w', round(d['value'],4), round(r['kernel_ms'],3), r.get('sm_clock_effective_mhz'), r.get('frac_per_clock'))
" >> $O/ab.txt; done
  done
done
cp /tmp/def.so paper_1909_01554_b200/libbmmgpu.so
cat $O/ab.txt
