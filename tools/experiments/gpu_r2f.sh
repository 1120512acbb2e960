#!/bin/bash
# Round 2, run F: level-shifted leaves (K2 fold mode) -- correctness and c2 / c4 A/B.
O=gpurun_out/r2f
mkdir -p $O
timeout 900 python -m pytest tests/test_alt_gpu.py tests/test_dropin.py tests/test_multidevice.py -m gpu -q -x > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt; tail -3 $O/tests.txt
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
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_c2_fold.csv \
    python bench.py --workload c2-gf2-altsi-65536 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-check > /dev/null 2>&1
python tools/launches.py $O/launches_c2_fold.csv > $O/launches_c2_fold.txt 2>&1; head -30 $O/launches_c2_fold.txt
