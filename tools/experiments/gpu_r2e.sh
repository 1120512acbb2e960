#!/bin/bash
# Round 2, run E: full GPU suite, out-of-core alt-si bench line at n = 2^19, first-call cost.
O=gpurun_out/r2e
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/tests_gpu.txt 2>&1; echo "rc=$?" >> $O/tests_gpu.txt; tail -3 $O/tests_gpu.txt
timeout 300 python microbench/first_call.py 65536 > $O/first_call.txt 2>&1; cat $O/first_call.txt
timeout 1500 python bench.py --workload c5-gf2-altooc-524288 --steps 2 --warmup 1 > $O/bench_c5_altooc.json 2> $O/bench_c5_altooc.err
tail -c 2500 $O/bench_c5_altooc.json; tail -5 $O/bench_c5_altooc.err
