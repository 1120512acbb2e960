# staged pageable copies after the persistent copy pool and the reshaping of contiguous copies
mkdir -p gpurun_out/st3
O=gpurun_out/st3
timeout 300 python microbench/staging.py 65536 > $O/s.txt 2>&1
timeout 300 python microbench/pageable.py 65536 >> $O/s.txt 2>&1
timeout 300 python microbench/pageable.py 131072 >> $O/s.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
cat $O/s.txt; tail -2 $O/pytest.log
