#!/bin/bash
# Round-2 closing pass on one box: GPU tests, smoke, bench, reference arm,
# then the measurement pass (tools/r2_measure.sh) under the same tag.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-r2f}
timeout 1700 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_tests.log 2>&1; echo tests=$? >> gpurun_out/${tag}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo smoke=$? >> gpurun_out/${tag}_smoke.log
timeout 500 python bench.py > gpurun_out/${tag}_bench.log 2>&1; echo bench=$? >> gpurun_out/${tag}_bench.log
timeout 500 python bench.py --impl reference > gpurun_out/${tag}_ref.log 2>&1; echo ref=$? >> gpurun_out/${tag}_ref.log
tail -n 2 gpurun_out/${tag}_tests.log; tail -n 2 gpurun_out/${tag}_smoke.log; grep '^{' gpurun_out/${tag}_bench.log | cut -c1-300; tail -n 1 gpurun_out/${tag}_ref.log
if [ -z "$SKIP_MEASURE" ]; then bash tools/r2_measure.sh ${tag}; fi
