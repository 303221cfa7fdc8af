set -x
I="python bench.py --interference --ranks 8"
timeout 300 $I --interference-impls sm,b2b,prelaunch_pcpy --gemm-priority high --interference-out gpurun_out/interf_prio.json > gpurun_out/interf_prio.log 2>&1
CECOLL_SM_TILES_PER_CTA=4 timeout 300 $I --interference-impls sm --gemm-priority high --interference-out gpurun_out/interf_prio_t4.json > gpurun_out/interf_prio_t4.log 2>&1
CECOLL_SM_TILES_PER_CTA=4 timeout 300 $I --interference-impls sm --interference-out gpurun_out/interf_t4.json > gpurun_out/interf_t4.log 2>&1
for g in 16 32 64; do CECOLL_SM_GRID=$g timeout 300 $I --interference-impls sm --interference-out gpurun_out/interf_grid$g.json > gpurun_out/interf_grid$g.log 2>&1; done
