#!/bin/bash
# A/B of block-product kernels with clock samples (dev helper).
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 500 > gpurun_out/ab_clocks.csv &
SMI=$!
for rep in 1 2; do
  python microbench/time_cubic.py ${1:-2,4,3} ${2:-8192,32768,65536}
done
kill $SMI
sort gpurun_out/ab_clocks.csv | uniq -c | sort -rn | head -5
