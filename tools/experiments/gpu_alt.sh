mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/alt_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/alt_pytest.log
for L in 12 13 11; do
  timeout 300 python bench.py --workload c2-gf2-altsi-65536 --leaf-log2 $L --no-cpu-baseline > gpurun_out/alt_c2_leaf$L.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/alt_launches_c2_leaf12.csv \
    python bench.py --workload c2-gf2-altsi-65536 --leaf-log2 12 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
cp paper_1909_01554_b200/libbmmgpu.so /tmp/new.so
cp build/v/g2.so paper_1909_01554_b200/libbmmgpu.so; echo "== g2" > gpurun_out/alt_g2.log; timeout 300 python microbench/time_leaf.py >> gpurun_out/alt_g2.log 2>&1
cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so
