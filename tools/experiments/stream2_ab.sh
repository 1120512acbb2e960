#!/bin/bash
# A/B of the two-level streamed fast path (default) against quadrant streaming
# (BMMGPU_ALT_STREAM_LEVELS=1) on configs[1] / configs[3], end to end from pinned buffers.
mkdir -p gpurun_out
out=gpurun_out/stream2_ab.txt
: > $out
timeout 600 python -m pytest tests/test_alt_gpu.py -q -x -m gpu 2>&1 | tail -3 >> $out
for rep in 1 2; do
  for lv in 2 1; do
    echo "levels=$lv" >> $out
    BMMGPU_ALT_STREAM_LEVELS=$lv timeout 300 python bench.py --workload c2-gf2-altsi-65536 --steps 10 --warmup 3 2>>gpurun_out/stream2_err.txt | tail -1 >> $out
  done
done
for lv in 2 1; do
  echo "levels=$lv c4" >> $out
  BMMGPU_ALT_STREAM_LEVELS=$lv timeout 600 python bench.py --workload c4-gf2-altsi-262144 --steps 3 --warmup 3 2>>gpurun_out/stream2_err.txt | tail -1 >> $out
done
