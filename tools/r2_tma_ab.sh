#!/bin/bash
# A/B of the TMA mover's shape policy (kernels.cu TmaPolicy): headline bench,
# SM-path plan sweep 64 KiB-256 MiB chunks, C++ latency 4 KiB-1 MiB.
#   POLICIES="name:ENV=.. ENV=..;name2:..." tools/r2_tma_ab.sh tag
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-tma_ab}
out=gpurun_out/${tag}.txt
: > $out
IFS=';' read -ra pols <<< "${POLICIES:-r1:CECOLL_TMA_ONEWAVE_RES=1 CECOLL_TMA_TILE=32768 CECOLL_TMA_WAVES=2;new:}"
for rep in ${REPS:-1 2}; do
for p in "${pols[@]}"; do
  name=${p%%:*}; envs=${p#*:}
  echo "== $name rep $rep ($envs)" >> $out
  env $envs timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-energy 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'], d['roofline']['frac'], d.get('parity_ok'))" >> $out 2>&1
  if [ $rep = 1 ]; then
    env $envs timeout 600 python bench.py --sweep --api plan --sweep-impls sm ${KINDS:+--sweep-kinds $KINDS} --sweep-sizes ${SIZES:-65536,262144,1048576,4194304,16777216,67108864,268435456} --sweep-out gpurun_out/${tag}_${name}_sweep.csv > /dev/null 2>&1
    python - gpurun_out/${tag}_${name}_sweep.csv >> $out <<'PY'
import csv, sys
for r in csv.DictReader(open(sys.argv[1])):
    print("sweep", r["collective"], r["size_bytes"], r["total_ns"], r["roofline_frac"], r["parity"])
PY
    [ -z "$NOLAT" ] && env $envs timeout 300 tools/latency 8 300 0 sm 2>&1 | grep -v "^#" >> $out
  fi
done
done
cat $out
