mkdir -p gpurun_out/diag
O=gpurun_out/diag
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python microbench/e2e_diag.py > $O/e2e_diag.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:cubic_umma2 -c 1 --csv python bench.py --workload c2-gf2-altsi-65536 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_c2_leaves.csv 2>/dev/null
timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline > $O/c2.log 2>&1
