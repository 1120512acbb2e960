mkdir -p gpurun_out/pc
O=gpurun_out/pc
cp paper_1909_01554_b200/libbmmgpu.so /tmp/new.so
for V in new pc4 new pc4; do
  if [ $V = new ]; then cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so; else cp build/v/$V.so paper_1909_01554_b200/libbmmgpu.so; fi
  echo "== $V"; timeout 300 python microbench/time_leaf.py 2048,4096
done > $O/ab.log 2>&1
cp build/v/pc4.so paper_1909_01554_b200/libbmmgpu.so
timeout 600 python -m pytest tests/test_cubic_gpu.py tests/test_alt_gpu.py -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
cp build/v/trace_pc4.so paper_1909_01554_b200/libbmmgpu.so
timeout 120 python microbench/trace_tiles.py 4096 64 > $O/trace.log 2>&1
cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so
