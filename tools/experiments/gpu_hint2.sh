mkdir -p gpurun_out/hint2
O=gpurun_out/hint2
cp paper_1909_01554_b200/libbmmgpu.so /tmp/new.so
for V in new h1rg12 h1rg16 h1rg24; do
  if [ $V = new ]; then cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so; else cp build/v/$V.so paper_1909_01554_b200/libbmmgpu.so; fi
  timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/c3_$V.log 2>&1
  timeout 600 python bench.py --workload c3-gf2-cubic-131072 --no-cpu-baseline --no-e2e > $O/c3g_$V.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:cubic_umma2 -c 1 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_$V.csv 2>/dev/null
done
cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so
