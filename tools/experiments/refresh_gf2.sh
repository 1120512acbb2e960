#!/bin/bash
# Refresh the GF(2) evidence after a K2 drain change: bench lines (configs[1], [3], scaled
# [4] with the independent spot check), the c2 launch list and one --set full leaf capture.
mkdir -p gpurun_out/ref2
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ref2/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/ref2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ref2/smoke.log 2>&1
O=gpurun_out/ref2
timeout 600 python bench.py --workload c2-gf2-altsi-65536 > $O/bench_c2_altsi.log 2>&1
timeout 600 python bench.py --workload c3-gf2-cubic-131072 --no-cpu-baseline > $O/bench_c3_gf2.log 2>&1
timeout 900 python bench.py --workload c4-gf2-altsi-262144 --steps 3 --no-cpu-baseline --e2e-steps 2 > $O/bench_c4_altsi.log 2>&1
timeout 1200 python bench.py --workload c5-gf2-ooc-524288 --steps 1 --warmup 1 --check > $O/bench_c5_gf2_ooc.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_c2_altsi.csv \
    python bench.py --workload c2-gf2-altsi-65536 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cubic_umma2 -s 1 -c 1 -o $O/full_umma2_c2_leaves \
    python bench.py --workload c2-gf2-altsi-65536 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/full_c2.log 2>&1
