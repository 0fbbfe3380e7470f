#!/bin/bash
mkdir -p gpurun_out/x
O=gpurun_out/x
for c in "0.5,0.5,3" "0.5,0.5,10" "0.3,0.7,3" "0.3,0.7,8" "0.7,0.3,3" "0.5,0.5,20"; do
  echo "== $c" >> $O/lpt.txt
  HNN_LPT_COST=$c timeout 300 python tools/plan_times.py x c3 2>&1 | grep -E 'tc2|sum' >> $O/lpt.txt
done
echo done
