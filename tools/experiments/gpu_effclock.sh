# effective SM clock (clock64 of the MMA lane / launch time) of K2 on a c3-size product and on leaves,
# with nvidia-smi clocks and power sampled alongside
mkdir -p gpurun_out/probe
O=gpurun_out/probe/effclock.txt
: > $O
cp paper_1909_01554_b200/libbmmgpu.so /tmp/libbmmgpu.orig.so
cp build/variants/libbmmgpu_probe.so paper_1909_01554_b200/libbmmgpu.so
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 100 > gpurun_out/probe/effclock_smi.csv &
P=$!
BMMGPU_UMMA_PROBE=0 timeout 300 python microbench/probe_leaf.py 131072 1 >> $O 2>&1
BMMGPU_UMMA_PROBE=64 timeout 300 python microbench/probe_leaf.py 131072 1 >> $O 2>&1
BMMGPU_UMMA_PROBE=0 timeout 300 python microbench/probe_leaf.py 4096 2401 >> $O 2>&1
kill $P
cp /tmp/libbmmgpu.orig.so paper_1909_01554_b200/libbmmgpu.so
cat $O
awk -F, '{split($2,a," "); if (a[1]+0 > 700) print}' gpurun_out/probe/effclock_smi.csv | sort | uniq -c | sort -rn | head
