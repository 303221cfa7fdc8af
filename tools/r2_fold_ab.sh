#!/bin/bash
# Prelaunch body A/B on one B200: the two-kernel body (gate_poll -> mover,
# default) against the folded single kernel (CECOLL_PRELAUNCH_FOLD=1), n = 8
# co-resident ranks, explicit plans, one stream (tools/latency).
cd "$(dirname "$0")/.."
tag=${1:-r2fold}
echo "body,api,impl,collective,size_bytes,device_us_b2b,device_us_isolated,host_us" > gpurun_out/${tag}.csv
for rep in 1 2; do
  for impl in prelaunch_b2b prelaunch_swap prelaunch_pcpy prelaunch_bcst; do
    timeout 120 tools/latency 8 300 0 $impl | grep -E "^plan," | grep -E ",(4096|65536|262144)," | sed "s/^/two_kernels,/"
    CECOLL_PRELAUNCH_FOLD=1 timeout 120 tools/latency 8 300 0 $impl | grep -E "^plan," | grep -E ",(4096|65536|262144)," | sed "s/^/folded,/"
  done
done >> gpurun_out/${tag}.csv
cat gpurun_out/${tag}.csv
