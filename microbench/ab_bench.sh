#!/bin/bash
# bench.py value / clocks with alternative builds of libbmmgpu.so (dev helper):
# ab_bench.sh "<bench args>" <lib>...
ARGS=$1; shift
for L in "$@"; do
  cp paper_1909_01554_b200/libbmmgpu.so /tmp/libbmmgpu.orig.so
  cp $L paper_1909_01554_b200/libbmmgpu.so
  echo "== $L"; python bench.py $ARGS --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({k: d.get(k) for k in ('value','ms_per_step','clocks')}), (d.get('e2e') or {}).get('value'))"
  cp /tmp/libbmmgpu.orig.so paper_1909_01554_b200/libbmmgpu.so
done
