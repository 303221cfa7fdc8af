#!/bin/bash
# A/B of the round-1 library (abtree/r01, built from 972628a) against the
# current one on the same box: C++ latency of the SM path and prelaunch.
cd "$(dirname "$0")/.."
tag=${1:-r2ab}
for rep in 1 2; do
  for impl in sm prelaunch_b2b prelaunch_swap; do
    timeout 120 abtree/r01/tools/latency 8 300 0 $impl | grep -E "^plan," | grep -E ",(4096|65536),"  | sed "s/^/r01,/"
    timeout 120 tools/latency 8 300 0 $impl | grep -E "^plan," | grep -E ",(4096|65536),"  | sed "s/^/r02,/"
    CECOLL_PRELAUNCH_FOLD=0 timeout 120 tools/latency 8 300 0 $impl | grep -E "^plan," | grep -E ",(4096|65536),"  | sed "s/^/r02nofold,/"
  done
done > gpurun_out/${tag}.csv
cat gpurun_out/${tag}.csv
