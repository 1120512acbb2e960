# quick round check on one B200: GPU tests, smoke, default bench, c2 bench (outputs under gpurun_out/q/)
mkdir -p gpurun_out/q
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/q/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/q/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/q/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/q/smoke.log
timeout 600 python bench.py > gpurun_out/q/bench_default.log 2>&1
timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline > gpurun_out/q/bench_c2.log 2>&1
tail -n 3 gpurun_out/q/*.log
