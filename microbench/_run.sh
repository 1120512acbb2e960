for L in build/v/l2p3.so build/v/l2p0.so build/v/rg16.so build/v/rg4.so cpasync; do
  cp paper_1909_01554_b200/libbmmgpu.so /tmp/orig.so
  if [ "$L" = cpasync ]; then export BMMGPU_UMMA_LOADER=cpasync; else cp $L paper_1909_01554_b200/libbmmgpu.so; fi
  echo "== $L"
  ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:umma2 -c 1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | grep -E "dram__|duration|hit_rate|per_second"
  unset BMMGPU_UMMA_LOADER
  cp /tmp/orig.so paper_1909_01554_b200/libbmmgpu.so
done
