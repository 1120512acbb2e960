# effective SM clock of K2 on a c3-size product: all operand stores (0), A stores removed after the
# first ring fill (128 = probe 4096), all stores removed after the first fill (64 = probe 2048)
mkdir -p gpurun_out/probe
O=gpurun_out/probe/effclock2.txt
: > $O
cp paper_1909_01554_b200/libbmmgpu.so /tmp/libbmmgpu.orig.so
cp build/variants/libbmmgpu_probe.so paper_1909_01554_b200/libbmmgpu.so
for P in 0 128 64 0 128; do
  BMMGPU_UMMA_PROBE=$P timeout 300 python microbench/probe_leaf.py 131072 1 >> $O 2>&1
done
cp /tmp/libbmmgpu.orig.so paper_1909_01554_b200/libbmmgpu.so
cat $O
