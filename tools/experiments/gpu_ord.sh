mkdir -p gpurun_out/ord
O=gpurun_out/ord
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2; do timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --e2e-steps 5 > $O/c2_$i.log 2>&1; done
timeout 900 python bench.py --workload c4-gf2-altsi-262144 --steps 3 --no-cpu-baseline --e2e-steps 2 > $O/c4.log 2>&1
