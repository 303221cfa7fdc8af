cd /root/repo
for pol in "p2:" "p1:CECOLL_TMA_TPC=1" "p4:CECOLL_TMA_TPC=4" "t8p2:CECOLL_TMA_TILE=8192" "t8p1:CECOLL_TMA_TILE=8192 CECOLL_TMA_TPC=1" "t32p2:CECOLL_TMA_TILE=32768" "f16:CECOLL_TMA_FAN_TILE=16384" "f4:CECOLL_TMA_FAN_TILE=4096"; do
  name=${pol%%:*}; envs=${pol#*:}
  env $envs timeout 300 python bench.py --sweep --api plan --ranks 2 --sweep-impls sm,pull,pcpy --sweep-sizes 1048576,4194304,16777216,67108864 --sweep-out gpurun_out/n2ab_${name}.csv > /dev/null 2>&1
done
