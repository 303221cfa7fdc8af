#!/bin/bash
# Round-2 probes: launch cost, PCIe duplex variants, prelaunch fold A/B, bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-r2p}
timeout 60 tools/launch_probe > gpurun_out/${tag}_launch_probe.txt 2>&1; echo "launch_probe rc=$?"
cat gpurun_out/${tag}_launch_probe.txt
timeout 300 python tools/pcie_probe4.py > gpurun_out/${tag}_pcie4.txt 2>&1; echo "pcie4 rc=$?"
head -12 gpurun_out/${tag}_pcie4.txt
for v in 1 0; do
  for impl in prelaunch_b2b prelaunch_swap sm; do
    CECOLL_PRELAUNCH_FOLD=$v timeout 120 tools/latency 8 300 0 $impl | grep -E "^plan," | grep -E ",(4096|65536|262144),"
  done | sed "s/^/fold=$v,/" >> gpurun_out/${tag}_fold_ab.csv
done
cat gpurun_out/${tag}_fold_ab.csv
timeout 600 python bench.py > gpurun_out/${tag}_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/${tag}_bench.log | head -c 3000
