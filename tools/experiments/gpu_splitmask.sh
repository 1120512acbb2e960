# streamed fast path end to end at n = 65536 for several split masks (bit i: child position i runs as 7 grandchildren)
mkdir -p gpurun_out/sm
O=gpurun_out/sm
: > $O/res.txt
for r in 1 2; do
for m in 0x41 0x01 0x03 0x43 0x61 0x63 0x40 0x00; do
  BMMGPU_ALT_SPLIT_MASK=$m timeout 200 python microbench/stream2_diag.py 65536 5 3 2>/dev/null | tail -n 1 | sed "s/^/$m /" >> $O/res.txt
done
done
cat $O/res.txt
