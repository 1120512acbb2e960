#!/bin/bash
# A/B of the pipelined in-core cubic path (row slices, default) against one in-order
# slice (BMMGPU_INCORE_SLICES=1) at configs[0], end to end from pinned buffers.
mkdir -p gpurun_out
out=gpurun_out/incore_ab.txt
: > $out
timeout 600 python -m pytest tests/test_cubic_gpu.py -q -x -m gpu 2>&1 | tail -3 >> $out
for rep in 1 2; do
  for sl in 4 1 2; do
    for wl in c1-bool-cubic-8192 c1-gf2-cubic-8192; do
      echo "slices=$sl $wl" >> $out
      BMMGPU_INCORE_SLICES=$sl timeout 300 python bench.py --workload $wl --steps 20 --warmup 5 2>>gpurun_out/incore_err.txt | tail -1 >> $out
    done
  done
done
