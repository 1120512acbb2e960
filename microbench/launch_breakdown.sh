#!/bin/bash
# Per-kernel device-time totals of one bench invocation (dev helper).
# usage: launch_breakdown.sh <tag> <bench args...>
TAG=$1; shift
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py "$@" --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python - "$TAG" <<'PY'
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(f"gpurun_out/launches_{sys.argv[1]}.csv")) if len(r) > 10 and r[0].isdigit()]
d = defaultdict(lambda: [0.0, 0])
for r in rows:
    d[r[4][:70]][0] += float(r[-1]); d[r[4][:70]][1] += 1
print(sys.argv[1])
for k, (v, c) in sorted(d.items(), key=lambda x: -x[1][0]):
    print(f"  {v/1e6:9.3f} ms  x{c:<5d} {k}")
PY
