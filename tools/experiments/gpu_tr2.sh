mkdir -p gpurun_out/tr2
O=gpurun_out/tr2
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2 3; do timeout 300 python bench.py --workload c1-bool-cubic-8192 --no-cpu-baseline > $O/c1b_$i.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:transpose --csv python bench.py --workload c2-gf2-altsi-65536 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_tr.csv 2>/dev/null
BMMGPU_TRANSPOSE_DIRECT=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:transpose --csv python bench.py --workload c2-gf2-altsi-65536 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_tr_direct.csv 2>/dev/null
