#!/bin/bash
# Round 2, run C: two overlapping accumulators in K2 -- correctness, leaf timing A/B against
# the one-accumulator build, tile trace, c2 bench.
O=gpurun_out/r2c
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 300 python microbench/race_k2.py 160 256 1024 > $O/race_small.txt 2>&1; tail -1 $O/race_small.txt
timeout 300 python microbench/race_k2.py 160 4096 4096 > $O/race_big.txt 2>&1; tail -1 $O/race_big.txt
timeout 900 python -m pytest tests/test_cubic_gpu.py tests/test_alt_gpu.py -m gpu -q -x > $O/tests.txt 2>&1; tail -2 $O/tests.txt
cp paper_1909_01554_b200/libbmmgpu.so /tmp/default.so
for rep in 1 2; do
  for v in default acc1; do
    if [ $v = default ]; then cp /tmp/default.so paper_1909_01554_b200/libbmmgpu.so; else cp build/variants/libbmmgpu_$v.so paper_1909_01554_b200/libbmmgpu.so; fi
    echo "== $v" >> $O/leaf_ab.txt
    timeout 300 python microbench/time_leaf.py 4096,2048 >> $O/leaf_ab.txt 2>&1
  done
done
for v in trace acc1trace; do
  cp build/variants/libbmmgpu_$v.so paper_1909_01554_b200/libbmmgpu.so
  timeout 120 python microbench/trace_tiles.py 4096 64 > $O/trace_$v.txt 2>&1
done
cp /tmp/default.so paper_1909_01554_b200/libbmmgpu.so
timeout 900 python bench.py --workload c2-gf2-altsi-65536 --steps 10 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err
tail -c 400 $O/bench_c2.json
cat $O/leaf_ab.txt
for tool in racecheck synccheck memcheck; do
  extra=""; [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 400 compute-sanitizer --tool $tool $extra --kernel-name regex=cubic_umma2 \
    python microbench/race_k2.py 40 256 1024 > $O/sanitizer_$tool.txt 2>&1
  echo "rc=$?" >> $O/sanitizer_$tool.txt; tail -3 $O/sanitizer_$tool.txt
done
for i in $(seq 1 20); do
  timeout 150 python -m pytest tests/test_multirank.py -q -m gpu -k alt_subinstance_deal 2>&1 | tail -1
done > $O/twoproc.txt
grep -c passed $O/twoproc.txt
