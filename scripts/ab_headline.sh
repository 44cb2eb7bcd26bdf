set -x
B="python bench.py --no-cpu-baseline --no-all-resident --no-checksum --lookahead 0 --steal-late 0 --steps 10"
for i in 1 2; do
  $B > gpurun_out/ab_default_$i.jsonl 2>/dev/null
  PS_SCHED_GRAPH=0 $B > gpurun_out/ab_nograph_$i.jsonl 2>/dev/null
  PS_HOST_LANE_SPLITRUN=1 $B > gpurun_out/ab_split_$i.jsonl 2>/dev/null
done
