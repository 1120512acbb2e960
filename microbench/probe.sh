#!/bin/bash
# Throughput of the persistent kernel's sides in isolation (dev helper; needs a
# -DBMMGPU_PROBE build, microbench/variant_lib.sh): probe 1 = producers only
# (no MMAs), probe 2 = MMAs only (no operand stores), results are garbage.
LIB=$1; N=${2:-32768,65536}
cp paper_1909_01554_b200/libbmmgpu.so /tmp/libbmmgpu.orig.so
cp $LIB paper_1909_01554_b200/libbmmgpu.so
for P in ${PROBES:-"" 1 2 4 8 9}; do
  echo "== probe '$P'"; BMMGPU_UMMA_PROBE=$P timeout 200 python microbench/time_cubic.py 2 $N | grep 'ring": 1'
done
cp /tmp/libbmmgpu.orig.so paper_1909_01554_b200/libbmmgpu.so
