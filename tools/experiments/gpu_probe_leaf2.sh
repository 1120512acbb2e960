# K2 expander-side costs on a batch of 4096^3 GF(2) leaves (probe build): no MMAs (1), + no proxy fence (17),
# + no Bt stores (33), both (49); MMAs with no fence (16), no Bt stores (32)
mkdir -p gpurun_out/probe
O=gpurun_out/probe/leaf2.txt
: > $O
cp paper_1909_01554_b200/libbmmgpu.so /tmp/libbmmgpu.orig.so
cp build/variants/libbmmgpu_probe.so paper_1909_01554_b200/libbmmgpu.so
for P in 0 1 17 33 49 16 32 0; do
  BMMGPU_UMMA_PROBE=$P timeout 120 python microbench/probe_leaf.py 4096 1200 >> $O 2>&1
done
BMMGPU_UMMA_PROBE=0 timeout 120 python microbench/probe_waits.py 32768 >> $O 2>&1
BMMGPU_UMMA_PROBE=1 timeout 120 python microbench/probe_waits.py 32768 >> $O 2>&1
cp /tmp/libbmmgpu.orig.so paper_1909_01554_b200/libbmmgpu.so
cat $O
