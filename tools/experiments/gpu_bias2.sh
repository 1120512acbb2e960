mkdir -p gpurun_out/bias2
O=gpurun_out/bias2
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
cp paper_1909_01554_b200/libbmmgpu.so /tmp/new.so
for V in new prev; do
  if [ $V = new ]; then cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so; else cp build/v/$V.so paper_1909_01554_b200/libbmmgpu.so; fi
  echo "== $V"; timeout 300 python microbench/time_leaf.py
done > $O/leaf.log 2>&1
cp build/v/trace_bias.so paper_1909_01554_b200/libbmmgpu.so
timeout 120 python microbench/trace_tiles.py 4096 64 > $O/trace.log 2>&1
cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so
timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline > $O/c2.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/c3.log 2>&1
