mkdir -p gpurun_out/pipe
O=gpurun_out/pipe
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for cfg in "16384 2 2" "65536 2 2" "65536 2 4" "65536 1 2"; do timeout 600 microbench/pipeline_bench $cfg >> $O/pipeline.log 2>&1; done
