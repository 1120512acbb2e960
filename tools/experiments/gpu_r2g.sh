#!/bin/bash
# Round 2, run G: level-shifted leaves with superstage units -- correctness, c2 / c4 A/B, first call.
O=gpurun_out/r2g
mkdir -p $O
timeout 900 python -m pytest tests/test_alt_gpu.py tests/test_capi.py -m gpu -q -x > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt; tail -3 $O/tests.txt
for rep in 1 2; do
  for f in 1 0; do
    BMMGPU_ALT_FOLD=$f timeout 900 python bench.py --workload c2-gf2-altsi-65536 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c2_fold$f.$rep.json 2> $O/bench_c2_fold$f.$rep.err
    python -c "import json,sys;d=json.loads(open('$O/bench_c2_fold$f.$rep.json').read().strip().splitlines()[-1]);print('fold=$f', d['value'], d['roofline']['kernel_ms'], d['ms_per_step'], d['parity']['ok'], d['clocks']['sm_mhz'])"
  done
done
for f in 1 0; do
  BMMGPU_ALT_FOLD=$f timeout 900 python bench.py --workload c4-gf2-altsi-262144 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c4_fold$f.json 2> $O/bench_c4_fold$f.err
  python -c "import json,sys;d=json.loads(open('$O/bench_c4_fold$f.json').read().strip().splitlines()[-1]);print('c4 fold=$f', d['value'], d['roofline']['kernel_ms'], d['ms_per_step'], d['parity']['ok'], d['clocks']['sm_mhz'])"
done
for m in none plain reserve; do timeout 300 python microbench/first_call.py 65536 $m; done > $O/first_call.txt 2>&1; cat $O/first_call.txt
