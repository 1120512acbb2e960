# K2 MMA side alone with valid operand data (probe 2048 = v 64: stores only while the ring first fills),
# with and without the fence (v 80), against the default kernel and the expanders alone (v 1)
mkdir -p gpurun_out/probe
O=gpurun_out/probe/leaf3.txt
: > $O
cp paper_1909_01554_b200/libbmmgpu.so /tmp/libbmmgpu.orig.so
cp build/variants/libbmmgpu_probe.so paper_1909_01554_b200/libbmmgpu.so
for P in 0 64 80 1 0 64; do
  BMMGPU_UMMA_PROBE=$P timeout 120 python microbench/probe_leaf.py 4096 1200 >> $O 2>&1
done
for P in 0 64; do
  BMMGPU_UMMA_PROBE=$P timeout 120 python microbench/probe_leaf.py 32768 2 >> $O 2>&1
done
cp /tmp/libbmmgpu.orig.so paper_1909_01554_b200/libbmmgpu.so
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv >> $O
cat $O
