timeout 300 python -m pytest tests/test_cubic_gpu.py tests/test_alt_gpu.py -q -x 2>&1 | tail -2
bash microbench/ab_lib.sh 8192,32768,65536 build/v/tma.so build/v/elect.so
