# gpu- vs system-scope per-CTA fence in fused epilogues (8 co-resident ranks, one stream per rank)
for v in 1 0 1 0; do
  echo "CECOLL_SYS_FENCE=$v"
  for i in sm prelaunch_pcpy prelaunch_b2b; do
    CECOLL_SYS_FENCE=$v timeout 120 tools/latency 8 300 1 $i | grep -E '^plan,' | grep -E ',(4096|65536|1048576),'
  done
  CECOLL_SYS_FENCE=$v timeout 120 tools/latency 8 300 1 sm | grep reduce_scatter | grep -E ',(4096|65536|1048576),'
done
