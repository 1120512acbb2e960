# full GPU suite + smoke on the current build, then the streamed c2 timeline (BMMGPU_ALT_TRACE)
mkdir -p gpurun_out/full
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/full/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/full/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/full/smoke.log
BMMGPU_ALT_TRACE=1 timeout 300 python microbench/stream2_diag.py 65536 3 3 > gpurun_out/full/trace_c2.txt 2>&1
tail -n 3 gpurun_out/full/*.log; tail -n 40 gpurun_out/full/trace_c2.txt
