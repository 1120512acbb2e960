mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/dram_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/dram_pytest.log
timeout 300 python microbench/dram_power.py > gpurun_out/dram_power.log 2>&1
timeout 300 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline > gpurun_out/dram_c2.log 2>&1
