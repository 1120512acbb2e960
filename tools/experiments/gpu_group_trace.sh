# Timeline of the overlapped leaf groups (BMMGPU_GROUP_TRACE), c2 device steps, 1 and 2 reserved pairs
O=gpurun_out/gt; mkdir -p $O
for ov in 1 2; do
  BMMGPU_GROUP_TRACE=1 BMMGPU_ALT_OVERLAP=$ov timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --no-check --no-e2e --steps 3 --warmup 3 > $O/c2_ov$ov.log 2>&1
done
grep groups $O/c2_ov1.log | tail -2; grep groups $O/c2_ov2.log | tail -2
