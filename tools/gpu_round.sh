set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
timeout 900 bash profiles/run_profiles.sh r01b c3-bool-cubic-131072 cubic_umma2 auto
tail -3 gpurun_out/*.log
