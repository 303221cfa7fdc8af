set -x
mkdir -p gpurun_out
for k in 1 2; do timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/soak_$k.log 2>&1; echo soak$k=$? >> gpurun_out/soak_$k.log; tail -3 gpurun_out/soak_$k.log; done
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --target-processes all python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "arm_and_trigger or other_device_signal_path or misrouted" > gpurun_out/memcheck_s3.txt 2>&1; tail -3 gpurun_out/memcheck_s3.txt
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python -m pytest tests/test_recorded.py -m gpu -q -x -k "caller_graph and (sm or pcpy)" > gpurun_out/racecheck_s3.txt 2>&1; tail -3 gpurun_out/racecheck_s3.txt
