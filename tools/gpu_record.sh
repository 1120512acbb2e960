# Round record: bench lines for every BASELINE config that fits one GPU, the reference arm,
# ncu launch lists and one --set full capture of each dominant kernel.
mkdir -p gpurun_out/rec
O=gpurun_out/rec
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_c3_bool.log 2>&1
timeout 600 python bench.py --impl reference > $O/bench_reference_c3.log 2>&1
timeout 600 python bench.py --workload c3-gf2-cubic-131072 --no-cpu-baseline > $O/bench_c3_gf2.log 2>&1
timeout 600 python bench.py --workload c2-gf2-altsi-65536 --e2e-steps 20 > $O/bench_c2_altsi.log 2>&1
timeout 600 python bench.py --workload c2-gf2-altsi-65536 --impl reference > $O/bench_reference_c2.log 2>&1
timeout 600 python bench.py --workload c1-gf2-cubic-8192 > $O/bench_c1_gf2.log 2>&1
timeout 600 python bench.py --workload c1-bool-cubic-8192 > $O/bench_c1_bool.log 2>&1
timeout 900 python bench.py --workload c4-gf2-altsi-262144 --steps 3 --no-cpu-baseline --e2e-steps 2 > $O/bench_c4_altsi.log 2>&1
timeout 900 python bench.py --workload c4-gf2-cubic-262144 --steps 2 --no-cpu-baseline --no-e2e > $O/bench_c4_cubic.log 2>&1
timeout 1200 python bench.py --workload c5-gf2-ooc-524288 --steps 1 --warmup 1 --check > $O/bench_c5_gf2_ooc.log 2>&1
timeout 1500 python bench.py --workload c5-gf2-altooc-524288 --steps 1 --warmup 1 --check > $O/bench_c5_gf2_altooc.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_c3_bool.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-check > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_c2_altsi.csv \
    python bench.py --workload c2-gf2-altsi-65536 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-check > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cubic_umma2 -s 1 -c 1 -o $O/full_umma2_c3_bool \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-check > $O/full_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cubic_umma2 -s 1 -c 1 -o $O/full_umma2_c2_leaves \
    python bench.py --workload c2-gf2-altsi-65536 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-check > $O/full_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:expand_pass -s 2 -c 1 -o $O/full_expand_c2 \
    python bench.py --workload c2-gf2-altsi-65536 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-check > $O/full_expand.log 2>&1
[ -x microbench/pipeline_bench ] || g++ -std=c++20 -O2 -I include microbench/pipeline_bench.cpp -o microbench/pipeline_bench -L paper_1909_01554_b200 -lbmm_b200 -lbmmgpu -Wl,-rpath,'$ORIGIN/../paper_1909_01554_b200' -lpthread
timeout 600 microbench/pipeline_bench 65536 2 2 > $O/pipeline.log 2>&1
tail -n 2 $O/*.log
