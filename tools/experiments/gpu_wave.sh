mkdir -p gpurun_out/wave
O=gpurun_out/wave
timeout 600 python -m pytest tests/test_cubic_gpu.py -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/c3_align.log 2>&1
BMMGPU_WAVE_ALIGN=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/c3_noalign.log 2>&1
cp paper_1909_01554_b200/libbmmgpu.so /tmp/new.so
for g in 8 32; do cp build/v/rg$g.so paper_1909_01554_b200/libbmmgpu.so; timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/c3_rg$g.log 2>&1; done
cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:cubic_umma2 -c 1 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_align.csv 2>/dev/null
BMMGPU_WAVE_ALIGN=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:cubic_umma2 -c 1 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_noalign.csv 2>/dev/null
