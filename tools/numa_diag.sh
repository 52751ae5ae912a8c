mkdir -p gpurun_out; o=gpurun_out/r01_v27_numa_diag.txt
{
nvidia-smi topo -m
ls /sys/devices/system/node/ | grep node
for n in /sys/devices/system/node/node*; do echo "$n $(cat $n/cpulist)"; done
python -c "
import torch; from paper_2211_00645_b200 import stream
p=torch.cuda.get_device_properties(0); print('pci', hex(p.pci_domain_id), hex(p.pci_bus_id), hex(p.pci_device_id)); print('gpu numa cpus', sorted(stream.gpu_numa_cpus(torch.device('cuda',0)) or [])[:4], len(stream.gpu_numa_cpus(torch.device('cuda',0)) or []))"
echo "== local (near_gpu)"
for i in 1 2; do timeout 200 python bench.py --config 3 --no-cpu-baseline | tail -1 | grep -o '"stacks_per_s": [0-9.]*\|"h2d_GBps": [0-9.]*\|"pinned_on_gpu_numa_node": [a-z]*' | tr '\n' ' '; echo; done
G=$(python -c "
import torch; from paper_2211_00645_b200 import stream; s=stream.gpu_numa_cpus(torch.device('cuda',0)); import os
allc=os.sched_getaffinity(0); other=sorted(allc-(s or set())); print(','.join(map(str,other)))")
echo "== other-node cpus: ${G:0:40}"
if [ -n "$G" ]; then for i in 1 2; do timeout 200 taskset -c $G python bench.py --config 3 --no-cpu-baseline | tail -1 | grep -o '"stacks_per_s": [0-9.]*\|"h2d_GBps": [0-9.]*\|"pinned_on_gpu_numa_node": [a-z]*' | tr '\n' ' '; echo; done; fi
} > $o 2>&1
cat $o
