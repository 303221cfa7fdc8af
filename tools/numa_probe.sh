#!/bin/bash
# Host topology of the GPU box and the PCIe duplex floor with the pinned
# buffers placed on each NUMA node (first touch follows the allocating
# thread's CPU affinity).
cd "$(dirname "$0")/.."
echo "== nproc $(nproc)"; lscpu | grep -E "^(CPU\(s\)|On-line|Model name|Socket|NUMA)"
command -v numactl >/dev/null && numactl -H
nvidia-smi topo -m 2>&1 | head -20
bus=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-F' 'a-f' | sed 's/^0000//; s/^/0000/')
echo "gpu bus $bus numa_node $(cat /sys/bus/pci/devices/${bus,,}/numa_node 2>/dev/null) local_cpulist $(cat /sys/bus/pci/devices/${bus,,}/local_cpulist 2>/dev/null)"
nvidia-smi -q | grep -A3 -i "link width\|PCIe Generation" | head -20
for n in /sys/devices/system/node/node*; do echo "$n cpus $(cat $n/cpulist)"; done
cpus_allowed=$(grep Cpus_allowed_list /proc/self/status)
echo "$cpus_allowed"
for n in /sys/devices/system/node/node*; do
  cl=$(cat $n/cpulist)
  echo "== pinned buffers on $(basename $n) (taskset -c $cl)"
  timeout 300 taskset -c "$cl" python tools/pcie_probe4.py 2>&1 | grep -v "^{" | head -8
done
