mkdir -p gpurun_out/f2
O=gpurun_out/f2
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python microbench/transform_ooc.py 13 $((12 << 30)) > $O/transform.log 2>&1
