#!/bin/bash
# Round 2, run D: full GPU suite (layout conversions, out-of-core alt tiles), layout
# throughput, the out-of-core alt-si bench line at n = 2^19, racecheck catalogue.
O=gpurun_out/r2d
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.total --format=csv > $O/smi.txt
free -g > $O/free.txt
timeout 1200 python -m pytest tests -m gpu -q -x > $O/tests_gpu.txt 2>&1; echo "rc=$?" >> $O/tests_gpu.txt; tail -3 $O/tests_gpu.txt
timeout 600 python microbench/layout_bench.py 131072 262144 > $O/layout_bench.txt 2>&1; cat $O/layout_bench.txt
timeout 1500 python bench.py --workload c5-gf2-altooc-524288 --steps 2 --warmup 1 > $O/bench_c5_altooc.json 2> $O/bench_c5_altooc.err
tail -c 1500 $O/bench_c5_altooc.json; tail -5 $O/bench_c5_altooc.err
timeout 400 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 100000 --kernel-name regex=cubic_umma2 \
    python microbench/race_k2.py 8 256 1024 > $O/sanitizer_racecheck_full.txt 2>&1
echo "rc=$?" >> $O/sanitizer_racecheck_full.txt
grep -o "hazard detected ([^)]*) at __shared__ 0x[0-9a-f]*" $O/sanitizer_racecheck_full.txt | awk '{print $NF}' | sort | uniq -c | sort -rn | head -20
