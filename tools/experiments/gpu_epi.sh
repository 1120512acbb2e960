mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cubic_gpu.py tests/test_alt_gpu.py -m gpu -x -q > gpurun_out/epi_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/epi_pytest.log
cp paper_1909_01554_b200/libbmmgpu.so /tmp/new.so
for V in new epi4; do
  if [ $V = new ]; then cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so; else cp build/v/$V.so paper_1909_01554_b200/libbmmgpu.so; fi
  echo "== $V"; timeout 300 python microbench/time_leaf.py; timeout 300 python microbench/time_cubic.py 2 32768 | head -1
done > gpurun_out/epi_ab.log 2>&1
cp build/v/trace8.so paper_1909_01554_b200/libbmmgpu.so
timeout 120 python microbench/trace_tiles.py 4096 64 > gpurun_out/epi_trace.log 2>&1
cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so
