# mxf4 pair MMA issue rate on K2-like operand values: burst and ~4 s under the power cap, clocks sampled
mkdir -p gpurun_out/ub
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 200 > gpurun_out/ub/sus_clocks.csv &
P=$!
timeout 120 ./microbench/ubench_sustained 4 > gpurun_out/ub/sustained.txt 2>&1
timeout 120 ./microbench/ubench_sustained 8 >> gpurun_out/ub/sustained.txt 2>&1
kill $P
cat gpurun_out/ub/sustained.txt; sort gpurun_out/ub/sus_clocks.csv | uniq -c | sort -rn | head -8
