# pageable staging: does GPU-local NUMA placement matter?  local_cpulist of the GPU, then pageable.py bound to it
mkdir -p gpurun_out/pg3
BUS=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-F' 'a-f' | sed 's/^0000//; s/^00000000/0000/')
echo "bus $BUS" > gpurun_out/pg3/info.txt
for d in /sys/bus/pci/devices/*; do if [ -f $d/local_cpulist ] && grep -qi "0x10de" $d/vendor 2>/dev/null && [ "$(cat $d/class)" = "0x030200" ]; then echo "$d $(cat $d/local_cpulist) numa $(cat $d/numa_node)" >> gpurun_out/pg3/info.txt; fi; done
lscpu | grep -i 'numa\|socket\|model name' >> gpurun_out/pg3/info.txt
CPUS=$(grep -m1 numa gpurun_out/pg3/info.txt | awk '{print $2}')
echo "cpus $CPUS" >> gpurun_out/pg3/info.txt
taskset -c $CPUS timeout 400 python microbench/pageable.py 65536 > gpurun_out/pg3/p65536_bound.txt 2>&1
cat gpurun_out/pg3/info.txt gpurun_out/pg3/p65536_bound.txt
