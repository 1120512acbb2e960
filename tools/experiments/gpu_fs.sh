mkdir -p gpurun_out/fs
O=gpurun_out/fs
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python microbench/time_leaf.py > $O/leaf.log 2>&1
cp paper_1909_01554_b200/libbmmgpu.so /tmp/new.so
cp build/v/trace_fs2.so paper_1909_01554_b200/libbmmgpu.so
timeout 120 python microbench/trace_tiles.py 4096 64 > $O/trace.log 2>&1
cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so
timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline > $O/c2.log 2>&1
timeout 900 python bench.py --workload c4-gf2-altsi-262144 --steps 3 --no-cpu-baseline --no-e2e > $O/c4.log 2>&1
