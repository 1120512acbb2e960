timeout 300 python -m pytest tests/test_cubic_gpu.py tests/test_alt_gpu.py -q -x 2>&1 | tail -2
bash microbench/ab_lib.sh 8192,32768,65536 build/v/grp48.so build/v/sst2.so build/v/sst3.so
cp build/v/probe.so paper_1909_01554_b200/libbmmgpu.so
for P in 0 1 2; do echo "probe $P"; BMMGPU_UMMA_PROBE=$P timeout 100 python microbench/probe_waits.py 32768; BMMGPU_UMMA_PROBE=$P timeout 100 python microbench/time_cubic.py 2 32768 | grep 'ring": 1'; done
