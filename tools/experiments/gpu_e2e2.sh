mkdir -p gpurun_out/e2e2
O=gpurun_out/e2e2
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python microbench/e2e_diag.py > $O/e2e_diag.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/c3.log 2>&1
