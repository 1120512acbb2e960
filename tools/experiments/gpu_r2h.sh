#!/bin/bash
# Round 2, run H: fold mode correctness (opt-in), operand ring of 2 stages (more fold units) A/B,
# first-call cost with bmmgpu_init.
O=gpurun_out/r2h
mkdir -p $O
timeout 900 python -m pytest tests/test_alt_gpu.py tests/test_capi.py -m gpu -q -x > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt; tail -3 $O/tests.txt
cp paper_1909_01554_b200/libbmmgpu.so /tmp/default.so
for v in default stages2; do
  if [ $v = default ]; then cp /tmp/default.so paper_1909_01554_b200/libbmmgpu.so; else cp build/variants/libbmmgpu_$v.so paper_1909_01554_b200/libbmmgpu.so; fi
  echo "== $v" >> $O/leaf.txt
  timeout 300 python microbench/time_leaf.py 4096,2048 >> $O/leaf.txt 2>&1
  for f in 0 1; do
    BMMGPU_ALT_FOLD=$f timeout 900 python bench.py --workload c2-gf2-altsi-65536 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c2_${v}_fold$f.json 2> $O/bench_c2_${v}_fold$f.err
    python -c "import json,sys;d=json.loads(open('$O/bench_c2_${v}_fold$f.json').read().strip().splitlines()[-1]);print('$v fold=$f', d['value'], d['roofline']['kernel_ms'], d['ms_per_step'], d['parity']['ok'], d['clocks']['sm_mhz'])"
  done
done
cp /tmp/default.so paper_1909_01554_b200/libbmmgpu.so
cat $O/leaf.txt
for m in none plain reserve; do timeout 300 python microbench/first_call.py 65536 $m; done > $O/first_call.txt 2>&1; cat $O/first_call.txt
