#!/bin/bash
# Round-2 measurement pass (one B200): latency tables, plan sweep with phase
# columns, reduce-scatter sweep, interference with SM budgets and host-resident
# copy-engine lanes, sync chain, ncu launch list + full capture of the bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-r2m}
run() { local name=$1; shift; local t0=$(date +%s); timeout "$@"; echo "== $name rc=$? $(( $(date +%s) - t0 ))s"; }
[ -z "$SKIP_LAT" ] && run lat_n8 300 tools/latency 8 300 0 > gpurun_out/${tag}_lat_n8.csv
[ -z "$SKIP_LAT" ] && run lat_n2 300 tools/latency 2 300 0 > gpurun_out/${tag}_lat_n2.csv
[ -z "$SKIP_SWEEP" ] && run sweep_n8 900 python bench.py --sweep --api plan --ranks 8 --sweep-out gpurun_out/${tag}_sweep_n8.csv > gpurun_out/${tag}_sweep_n8.log 2>&1
[ -z "$SKIP_SWEEP" ] && run sweep_n2 900 python bench.py --sweep --api plan --ranks 2 --sweep-out gpurun_out/${tag}_sweep_n2.csv > gpurun_out/${tag}_sweep_n2.log 2>&1
[ -z "$SKIP_INTF" ] && run interference 900 python bench.py --interference --gemm-iters 100 --interference-out gpurun_out/${tag}_interference.json > gpurun_out/${tag}_interference.log 2>&1
[ -z "$SKIP_SYNC" ] && run sync_chain 600 python bench.py --sync-chain --sync-out gpurun_out/${tag}_sync_chain.json > gpurun_out/${tag}_sync_chain.log 2>&1
[ -z "$SKIP_RS" ] && run sweep_rs 600 python bench.py --sweep-rs --sweep-out gpurun_out/${tag}_sweep_rs.csv > gpurun_out/${tag}_sweep_rs.log 2>&1
if [ -z "$SKIP_NCU" ]; then
  run ncu_launches 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 3 --warmup 3 --no-energy --no-cpu-baseline --e2e-steps 4 > gpurun_out/${tag}_ncu_bench.log 2>&1
  run ncu_full 900 ncu --set full --clock-control none --import-source on -k regex:tma_items -s 6 -c 1 -o gpurun_out/${tag}_items python bench.py --steps 3 --warmup 3 --no-energy --no-cpu-baseline --e2e-steps 4 > gpurun_out/${tag}_ncu_full.log 2>&1
fi
ls -la gpurun_out | grep ${tag}
