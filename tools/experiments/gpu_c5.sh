mkdir -p gpurun_out/c5
O=gpurun_out/c5
free -g > $O/free.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 1200 python bench.py --workload c5-gf2-ooc-524288 --steps 1 --warmup 1 --check > $O/c5_gf2.log 2>&1
timeout 1200 python bench.py --workload c5-bool-ooc-524288 --steps 1 --warmup 1 > $O/c5_bool.log 2>&1
