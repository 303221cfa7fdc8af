# Round-2 validation on one fresh box (same steps as final_validation_r01.sh): GPU tests, smoke, bench, reference arm, launch list of the bench under ncu.
mkdir -p gpurun_out
timeout 1700 python -m pytest tests -m gpu -q -x > gpurun_out/v2_tests.log 2>&1; echo tests=$? >> gpurun_out/v2_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v2_smoke.log 2>&1; echo smoke=$? >> gpurun_out/v2_smoke.log
timeout 500 python bench.py > gpurun_out/v2_bench.log 2>&1; echo bench=$? >> gpurun_out/v2_bench.log
timeout 500 python bench.py --impl reference > gpurun_out/v2_ref.log 2>&1; echo ref=$? >> gpurun_out/v2_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/v2_ncu_bench.log 2>&1; echo ncu=$? >> gpurun_out/v2_ncu_bench.log
tail -n 2 gpurun_out/v2_tests.log; tail -n 2 gpurun_out/v2_smoke.log; tail -c 300 gpurun_out/v2_bench.log; tail -c 200 gpurun_out/v2_ref.log; tail -n 1 gpurun_out/v2_ncu_bench.log
