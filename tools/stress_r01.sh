# Long back-to-back stress of every implementation (tools/b2b_stress.py), both signal paths.
for m in plain force; do
  for i in sm pcpy b2b bcst prelaunch_bcst prelaunch_pcpy hybrid pull; do
    timeout 200 python tools/b2b_stress.py $i 30 $m allgather 2>&1 | tail -n 2
  done
  for i in sm swap prelaunch_swap hybrid pull prelaunch_b2b; do
    timeout 200 python tools/b2b_stress.py $i 30 $m alltoall 2>&1 | tail -n 2
  done
done
