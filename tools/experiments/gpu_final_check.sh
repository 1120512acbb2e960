# Final check of HEAD: GPU suite, smoke, default bench, c2 / c4 / c5-alt lines with parity
O=gpurun_out/fc; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_c3_bool.log 2>&1
timeout 600 python bench.py --workload c2-gf2-altsi-65536 --e2e-steps 20 --no-cpu-baseline > $O/bench_c2_altsi.log 2>&1
timeout 900 python bench.py --workload c4-gf2-altsi-262144 --steps 3 --no-cpu-baseline --e2e-steps 2 > $O/bench_c4_altsi.log 2>&1
timeout 1500 python bench.py --workload c5-gf2-altooc-524288 --steps 1 --warmup 1 --check > $O/bench_c5_gf2_altooc.log 2>&1
tail -n 2 $O/pytest_gpu.log $O/smoke.log
python tools/summarize_rec.py $O
