#!/bin/bash
mkdir -p gpurun_out/s
O=gpurun_out/s
for n in 2 4 8; do
  for r in 0 $((n-1)); do
    timeout 300 python bench.py --shard $r/$n --no-cpu --steps 20 --warmup 5 > $O/shard_${r}_of_${n}.json 2> $O/shard_${r}_of_${n}.err
  done
done
timeout 300 python tools/plan_times.py x c3 > $O/plan_full.txt 2>&1
echo done
