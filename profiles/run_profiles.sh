#!/bin/bash
# Reproduces the committed profiles (run under gpurun on one B200).
#   launches_<tag>.csv : every kernel launch of a short bench run with its device time
#                        (ncu --metrics gpu__time_duration.sum --clock-control none)
#   full_<tag>.ncu-rep : one ncu --set full capture of the product kernel
set -u
TAG=${1:-r01}
WL=${2:-c3-bool-cubic-131072}
KREGEX=${3:-cubic_}
KER=${4:-auto}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --workload $WL --kernel $KER --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
    > gpurun_out/launches_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s 1 -c 1 -o gpurun_out/full_${TAG} \
    python bench.py --workload $WL --kernel $KER --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
    > gpurun_out/full_${TAG}.log 2>&1
