mkdir -p gpurun_out
free -g > gpurun_out/free.txt; nproc >> gpurun_out/free.txt; lscpu | grep "Model name" >> gpurun_out/free.txt
for L in 12 13 11; do
  timeout 300 python bench.py --workload c2-gf2-altsi-65536 --leaf-log2 $L --no-cpu-baseline --no-e2e > gpurun_out/c2_leaf$L.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_leaf$L.csv \
    python bench.py --workload c2-gf2-altsi-65536 --leaf-log2 $L --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
