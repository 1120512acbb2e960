#!/bin/bash
# Time the default kernel with alternative builds of libbmmgpu.so (dev helper):
# ab_lib.sh <n list> <lib>...
N=$1; shift
for L in "$@"; do
  cp paper_1909_01554_b200/libbmmgpu.so /tmp/libbmmgpu.orig.so
  cp $L paper_1909_01554_b200/libbmmgpu.so
  echo "== $L"; timeout 200 python microbench/time_cubic.py 2 $N | grep 'ring": 1'
  cp /tmp/libbmmgpu.orig.so paper_1909_01554_b200/libbmmgpu.so
done
