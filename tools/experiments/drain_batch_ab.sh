#!/bin/bash
# A/B of a K2 epilogue drain variant (new build) against build/v/old.so --

mkdir -p gpurun_out
O=gpurun_out/drain_ab.txt
: > $O
timeout 600 python -m pytest tests/test_cubic_gpu.py tests/test_alt_gpu.py -m gpu -x -q 2>&1 | tail -2 >> $O
cp paper_1909_01554_b200/libbmmgpu.so /tmp/new.so
for rep in 1 2; do
  for v in old new; do
    if [ $v = old ]; then cp build/v/old.so paper_1909_01554_b200/libbmmgpu.so; else cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so; fi
    echo "== $v leaf" >> $O; timeout 300 python microbench/time_leaf.py 4096,2048 >> $O 2>&1
    echo "== $v c2" >> $O; timeout 300 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 >> $O
    echo "== $v c3gf2" >> $O; timeout 300 python bench.py --workload c3-gf2-cubic-131072 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 >> $O
  done
done
cp /tmp/new.so paper_1909_01554_b200/libbmmgpu.so
