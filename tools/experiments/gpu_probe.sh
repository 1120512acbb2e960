mkdir -p gpurun_out/probe
O=gpurun_out/probe
cp build/v/probe_drain.so paper_1909_01554_b200/libbmmgpu.so
timeout 120 python microbench/trace_tiles.py 4096 64 > $O/trace_probe.log 2>&1
timeout 120 python microbench/time_leaf.py 4096 > $O/leaf_probe.log 2>&1
