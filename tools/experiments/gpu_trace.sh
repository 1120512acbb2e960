mkdir -p gpurun_out
cp build/v/trace.so paper_1909_01554_b200/libbmmgpu.so
for L in 4096 2048 8192; do timeout 120 python microbench/trace_tiles.py $L 64; done > gpurun_out/trace_tiles.log 2>&1
