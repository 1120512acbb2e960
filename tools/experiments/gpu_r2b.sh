#!/bin/bash
# Round 2, run B: full GPU suite + smoke, default bench (c3) and c2 with parity, K2 race investigation.
O=gpurun_out/r2b
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
lscpu | head -20 > $O/lscpu.txt
timeout 900 python -m pytest tests -m gpu -q -x > $O/tests_gpu.txt 2>&1; echo "rc=$?" >> $O/tests_gpu.txt
tail -3 $O/tests_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err; tail -c 1500 $O/bench_c3.json
timeout 900 python bench.py --workload c2-gf2-altsi-65536 --steps 10 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err
tail -c 600 $O/bench_c2.json
# race investigation
cp paper_1909_01554_b200/libbmmgpu.so /tmp/orig.so
for v in 2 1 0; do
  cp build/variants/libbmmgpu_pack16_$v.so paper_1909_01554_b200/libbmmgpu.so
  for tool in racecheck synccheck; do
    extra=""; [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout 300 compute-sanitizer --tool $tool $extra --kernel-name regex:cubic_umma2 \
      python microbench/race_k2.py 40 256 1024 > $O/race_${tool}_v$v.txt 2>&1
    echo "rc=$?" >> $O/race_${tool}_v$v.txt
  done
done
for v in 2 1 0; do
  cp build/variants/libbmmgpu_pack16_$v.so paper_1909_01554_b200/libbmmgpu.so
  for i in $(seq 1 20); do
    timeout 150 python -m pytest tests/test_multirank.py -q -m gpu -k alt_subinstance_deal 2>&1 | tail -1
  done > $O/race_twoproc_v$v.txt
  timeout 300 python microbench/race_k2.py 160 4096 4096 > $O/race_k2_big_v$v.txt 2>&1
done
cp /tmp/orig.so paper_1909_01554_b200/libbmmgpu.so
grep -c passed $O/race_twoproc_v*.txt
