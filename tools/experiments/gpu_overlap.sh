# Overlapped leaf groups (alt.cu, BMMGPU_ALT_OVERLAP = CTA pairs left to the passes; 0 = off):
# alt GPU tests, then the c2 / c4 benches alternated over the setting on one box.
O=gpurun_out/ov; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests/test_alt_gpu.py tests/test_multidevice.py -m gpu -x -q > $O/pytest_alt.log 2>&1; echo "rc=$?" >> $O/pytest_alt.log
for r in 1 2; do
  for ov in 0 2 1 4; do
    echo "== ov=$ov" >> $O/c2.txt
    BMMGPU_ALT_OVERLAP=$ov timeout 600 python bench.py --workload c2-gf2-altsi-65536 --no-cpu-baseline --no-check --e2e-steps 10 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],3), round(d['ms_per_step'],2), round(d['e2e']['value'],3), r.get('sm_clock_effective_mhz'), round(r.get('kernel_share_of_step',0),3))" >> $O/c2.txt 2>&1
  done
done
for ov in 0 2; do
  echo "== ov=$ov" >> $O/c4.txt
  BMMGPU_ALT_OVERLAP=$ov timeout 900 python bench.py --workload c4-gf2-altsi-262144 --steps 2 --no-cpu-baseline --no-check --e2e-steps 1 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],3), round(d['ms_per_step'],2), round(d['e2e']['value'],3), r.get('sm_clock_effective_mhz'))" >> $O/c4.txt 2>&1
done
tail -n 3 $O/pytest_alt.log; cat $O/c2.txt $O/c4.txt
