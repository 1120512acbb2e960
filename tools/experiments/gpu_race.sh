#!/bin/bash
# K2 race investigation (round 2): sanitizer runs on the three GF(2) drain variants and
# repeated two-process tile tests.  Outputs under gpurun_out/race_*.
mkdir -p gpurun_out
cp paper_1909_01554_b200/libbmmgpu.so /tmp/orig.so
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/race_smi.txt
timeout 120 python microbench/race_k2.py > gpurun_out/race_plain.txt 2>&1; echo "plain rc=$?" >> gpurun_out/race_plain.txt
for v in 2 1 0; do
  cp build/variants/libbmmgpu_pack16_$v.so paper_1909_01554_b200/libbmmgpu.so
  for tool in racecheck synccheck memcheck; do
    extra=""; [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout 400 compute-sanitizer --tool $tool $extra --kernel-name regex:cubic_umma2 \
      python microbench/race_k2.py 40 256 1024 > gpurun_out/race_${tool}_v$v.txt 2>&1
    echo "rc=$?" >> gpurun_out/race_${tool}_v$v.txt
  done
done
for v in 2 0 1; do
  cp build/variants/libbmmgpu_pack16_$v.so paper_1909_01554_b200/libbmmgpu.so
  n=30; [ $v = 2 ] && n=50
  for i in $(seq 1 $n); do
    timeout 150 python -m pytest tests/test_multirank.py -q -m gpu -k alt_subinstance_deal 2>&1 | tail -1
  done > gpurun_out/race_twoproc_v$v.txt
done
cp /tmp/orig.so paper_1909_01554_b200/libbmmgpu.so
