# K3 transpose: XOR-swizzled shared layout (default) vs the round-1 padded layout (oldtr variant); transpose tests
mkdir -p gpurun_out/tr
O=gpurun_out/tr
timeout 600 python -m pytest tests/test_cubic_gpu.py tests/test_alt_gpu.py -m gpu -q -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
cp paper_1909_01554_b200/libbmmgpu.so /tmp/new.so
: > $O/ab.txt
for i in 1 2; do
  cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so; echo "== swizzled" >> $O/ab.txt; timeout 120 python microbench/time_transpose.py >> $O/ab.txt 2>&1
  cp build/variants/libbmmgpu_oldtr.so paper_1909_01554_b200/libbmmgpu.so; echo "== padded (r1)" >> $O/ab.txt; timeout 120 python microbench/time_transpose.py >> $O/ab.txt 2>&1
done
cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so
timeout 300 ncu --set full --clock-control none -k regex:transpose_staged -s 3 -c 1 -o $O/full_transpose python microbench/time_transpose.py 65536 > /dev/null 2>&1
tail -2 $O/pytest.log; cat $O/ab.txt
