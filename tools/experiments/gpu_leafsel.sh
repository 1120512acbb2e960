mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cubic_gpu.py tests/test_alt_gpu.py -m gpu -x -q > gpurun_out/ls_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ls_pytest.log
timeout 300 python microbench/time_leaf.py > gpurun_out/ls_leaf.log 2>&1
for L in 12 13; do
  timeout 300 python bench.py --workload c2-gf2-altsi-65536 --leaf-log2 $L --no-cpu-baseline --no-e2e > gpurun_out/ls_c2_$L.log 2>&1
  timeout 600 python bench.py --workload c4-gf2-altsi-262144 --leaf-log2 $L --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/ls_c4_$L.log 2>&1
done
cp paper_1909_01554_b200/libbmmgpu.so /tmp/new.so; cp build/v/trace4.so paper_1909_01554_b200/libbmmgpu.so
timeout 120 python microbench/trace_tiles.py 4096 64 > gpurun_out/ls_trace.log 2>&1
cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so
