#!/bin/bash
mkdir -p gpurun_out
L=paper_2408_01331_b200/_lib/variants
for i in 1 2; do
echo "== default" >> gpurun_out/ring_plan.txt
timeout 300 python tools/plan_times.py x c3 2>&1 | grep -E 'tc2|sum' >> gpurun_out/ring_plan.txt
echo "== r3" >> gpurun_out/ring_plan.txt
timeout 300 python tools/plan_times.py $L/r3/libhnn_b200.so c3 2>&1 | grep -E 'tc2|sum' >> gpurun_out/ring_plan.txt
done
timeout 300 python tools/tc2_trace.py $L/r3trace/libhnn_b200.so c3 > gpurun_out/r3_trace.txt 2>&1
echo done
