mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/bias_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/bias_pytest.log
timeout 300 python microbench/time_leaf.py > gpurun_out/bias_leaf.log 2>&1
for L in 12 13; do timeout 300 python bench.py --workload c2-gf2-altsi-65536 --leaf-log2 $L --no-cpu-baseline > gpurun_out/bias_c2_$L.log 2>&1; done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bias_c3.log 2>&1
