mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/alt2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/alt2_pytest.log
timeout 300 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline > gpurun_out/alt2_c2.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/alt2_launches.csv \
    python bench.py --workload c2-gf2-altsi-65536 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
cp paper_1909_01554_b200/libbmmgpu.so /tmp/new.so
cp build/v/cv1.so paper_1909_01554_b200/libbmmgpu.so
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/alt2_launches_cv1.csv \
    python bench.py --workload c2-gf2-altsi-65536 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so
