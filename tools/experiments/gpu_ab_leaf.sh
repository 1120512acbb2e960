mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_cubic_gpu.py tests/test_alt_gpu.py -m gpu -x -q > gpurun_out/ab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab_pytest.log
cp paper_1909_01554_b200/libbmmgpu.so /tmp/new.so
{
echo "== old"; cp build/v/old.so paper_1909_01554_b200/libbmmgpu.so; timeout 300 python microbench/time_leaf.py
cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so
echo "== new (adaptive sleep)"; timeout 300 python microbench/time_leaf.py
for S in 0 32 128 512; do echo "== new sleep $S"; BMMGPU_EPI_SLEEP_NS=$S timeout 300 python microbench/time_leaf.py; done
} > gpurun_out/ab_leaf.log 2>&1
timeout 300 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --no-e2e > gpurun_out/ab_c2.log 2>&1
timeout 300 python bench.py --workload c2-gf2-altsi-65536 --leaf-log2 13 --no-cpu-baseline --no-e2e >> gpurun_out/ab_c2.log 2>&1
