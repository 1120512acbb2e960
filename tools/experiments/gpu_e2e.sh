mkdir -p gpurun_out/e2e
O=gpurun_out/e2e
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --no-cpu-baseline > $O/c3.log 2>&1
timeout 600 python bench.py --workload c3-gf2-cubic-131072 --no-cpu-baseline > $O/c3g.log 2>&1
timeout 1200 python bench.py --workload c5-gf2-ooc-524288 --steps 1 --warmup 1 > $O/c5_gf2.log 2>&1
