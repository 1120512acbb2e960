# K2 on a batch of 4096^3 GF(2) leaves: default build, then the probe build with each isolation probe
mkdir -p gpurun_out/probe
O=gpurun_out/probe/leaf.txt
echo "== default" > $O
python microbench/probe_leaf.py 4096 1200 >> $O 2>&1
python microbench/probe_leaf.py 2048 4201 >> $O 2>&1
cp paper_1909_01554_b200/libbmmgpu.so /tmp/libbmmgpu.orig.so
cp build/variants/libbmmgpu_probe.so paper_1909_01554_b200/libbmmgpu.so
for P in 0 1 2 4 8 9; do
  echo "== probe $P" >> $O
  BMMGPU_UMMA_PROBE=$P timeout 120 python microbench/probe_leaf.py 4096 1200 >> $O 2>&1
done
cp /tmp/libbmmgpu.orig.so paper_1909_01554_b200/libbmmgpu.so
cat $O
