#!/bin/bash
# Soak of the default GF(2) drain (BMMGPU_GF2_PACK16=1, in-register shuffle) under concurrency:
# the two-rank alt sub-instance deal (two processes sharing one GPU, parity checked against
# the cubic product) R times over leaf sizes 2^9..2^12 and both K2 loaders, then the
# single-process race batch at several leaf sizes.  Output: gpurun_out/soak/soak.txt
R=${1:-100}
mkdir -p gpurun_out/soak
out=gpurun_out/soak/soak.txt
: > $out
pass=0; fail=0
declare -A P F
for i in $(seq 1 $R); do
  leaf=$((9 + i % 4))
  if (( (i / 4) % 2 )); then ld=cpasync; else ld=tma; fi
  key="leaf$leaf-$ld"
  r=$(BMM_DIST_BACKEND=gloo BMMGPU_UMMA_LOADER=$ld timeout 300 python -m torch.distributed.run --nnodes=1 \
      --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600 + i % 50)) bench.py --gpus 2 \
      --workload c4s-gf2-altsi-16384 --leaf-log2 $leaf --steps 3 --warmup 3 2>/dev/null | grep '^{' | head -1)
  ok=$(echo "$r" | python -c 'import json,sys
try:
    d=json.loads(sys.stdin.read()); print(int(d["parity"]["ok"] is True and d["parity"]["slab_equals_cubic_product"] is True))
except Exception: print(0)')
  if [ "$ok" = 1 ]; then pass=$((pass+1)); P[$key]=$((${P[$key]:-0}+1)); else fail=$((fail+1)); F[$key]=$((${F[$key]:-0}+1)); echo "run $i $key FAILED: $r" >> $out; fi
done
echo "# two-rank alt sub-instance deal (c4s-gf2-altsi-16384, 2 processes on one GPU), default drain" >> $out
for k in "${!P[@]}" "${!F[@]}"; do echo "$k"; done | sort -u | while read k; do
  echo "$k: ${P[$k]:-0} passed, ${F[$k]:-0} failed" >> $out; done
echo "total: $pass passed, $fail failed of $R" >> $out
echo "# single process race batch (microbench/race_k2.py batch L K), both loaders" >> $out
for ld in tma cpasync; do for L in 256 512 1024 2048 4096; do
  echo "$ld: $(BMMGPU_UMMA_LOADER=$ld timeout 300 python microbench/race_k2.py 160 $L $L 2>&1 | tail -1)" >> $out
done; done
cat $out
