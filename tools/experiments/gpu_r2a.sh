#!/bin/bash
# Round 2, run A: new GPU tests, GF(2) drain A/B (32- vs 64-column TMEM loads), bench lines with parity.
mkdir -p gpurun_out/r2a
O=gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 900 python -m pytest tests/test_multidevice.py tests/test_alt_gpu.py tests/test_cubic_gpu.py tests/test_dropin.py tests/test_capi.py -m gpu -q -x > $O/tests_new.txt 2>&1
tail -5 $O/tests_new.txt
cp paper_1909_01554_b200/libbmmgpu.so /tmp/default.so
for v in trace32 trace64; do
  cp build/variants/libbmmgpu_$v.so paper_1909_01554_b200/libbmmgpu.so
  timeout 120 python microbench/trace_tiles.py 4096 64 > $O/trace_$v.txt 2>&1
done
for rep in 1 2; do
  for v in default drain64; do
    if [ $v = default ]; then cp /tmp/default.so paper_1909_01554_b200/libbmmgpu.so; else cp build/variants/libbmmgpu_$v.so paper_1909_01554_b200/libbmmgpu.so; fi
    echo "== $v" >> $O/leaf_ab.txt
    timeout 300 python microbench/time_leaf.py 4096,2048 >> $O/leaf_ab.txt 2>&1
  done
done
cp build/variants/libbmmgpu_drain64.so paper_1909_01554_b200/libbmmgpu.so
timeout 300 python microbench/race_k2.py 160 256 1024 > $O/race_k2_drain64.txt 2>&1
timeout 300 python microbench/race_k2.py 160 4096 4096 >> $O/race_k2_drain64.txt 2>&1
cp /tmp/default.so paper_1909_01554_b200/libbmmgpu.so
timeout 900 python bench.py --workload c2-gf2-altsi-65536 --steps 10 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
tail -c 3000 $O/bench_c3.json
