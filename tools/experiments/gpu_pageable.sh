# pageable (std::vector-like) vs pinned host buffers through the C ABI after the staging changes
mkdir -p gpurun_out/pg2
nproc > gpurun_out/pg2/nproc.txt
timeout 400 python microbench/pageable.py 65536 > gpurun_out/pg2/p65536.txt 2>&1
timeout 400 python microbench/pageable.py 131072 > gpurun_out/pg2/p131072.txt 2>&1
timeout 600 python -m pytest tests/test_cubic_gpu.py -m gpu -q -k "pageable or out_of_core or concurrent" > gpurun_out/pg2/pytest.log 2>&1; echo rc=$? >> gpurun_out/pg2/pytest.log
cat gpurun_out/pg2/nproc.txt gpurun_out/pg2/p*.txt; tail -2 gpurun_out/pg2/pytest.log
