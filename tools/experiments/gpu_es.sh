mkdir -p gpurun_out/es
O=gpurun_out/es
cp paper_1909_01554_b200/libbmmgpu.so /tmp/new.so
for V in new es0 es128; do
  if [ $V = new ]; then cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so; else cp build/v/$V.so paper_1909_01554_b200/libbmmgpu.so; fi
  echo "== $V"; timeout 300 python microbench/time_leaf.py; timeout 300 python microbench/time_cubic.py 2 32768 2>/dev/null | head -1
done > $O/ab.log 2>&1
cp build/v/trace_es.so paper_1909_01554_b200/libbmmgpu.so
timeout 120 python microbench/trace_tiles.py 4096 64 > $O/trace.log 2>&1
cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so
timeout 600 python -m pytest tests/test_cubic_gpu.py -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/c3.log 2>&1
