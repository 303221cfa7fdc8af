#!/bin/bash
# Round-2 GPU check: every GPU test file on its own (a hang costs only that
# file), smoke, C++ latency table (n=8, one stream).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-r2}
files=${FILES:-$(ls tests/test_*.py)}
: > gpurun_out/${tag}_tests.log
for f in $files; do
  start=$(date +%s)
  timeout ${FILE_TIMEOUT:-420} python -u -m pytest "$f" -q -m gpu -x -p no:cacheprovider > gpurun_out/${tag}_one.log 2>&1
  rc=$?
  echo "== $f rc=$rc $(( $(date +%s) - start ))s $(tail -1 gpurun_out/${tag}_one.log)" | tee -a gpurun_out/${tag}_tests.log
  if [ $rc -ne 0 ] && [ $rc -ne 5 ]; then tail -40 gpurun_out/${tag}_one.log >> gpurun_out/${tag}_tests.log; fi
done
if [ -z "$SKIP_SMOKE" ]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke_rc=$?"
fi
if [ -z "$SKIP_LAT" ]; then
  timeout 600 tools/latency 8 300 0 ${LAT_FILTER:-} > gpurun_out/${tag}_lat_n8.csv 2>&1; echo "lat_rc=$?"
fi
