mkdir -p gpurun_out/hint
O=gpurun_out/hint
timeout 600 python -m pytest tests/test_cubic_gpu.py -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
cp paper_1909_01554_b200/libbmmgpu.so /tmp/new.so
for V in new hint1 hint2 rg9; do
  if [ $V = new ]; then cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so; else cp build/v/$V.so paper_1909_01554_b200/libbmmgpu.so; fi
  timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/c3_$V.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:cubic_umma2 -c 1 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_$V.csv 2>/dev/null
done
cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so
timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline > $O/c2.log 2>&1
