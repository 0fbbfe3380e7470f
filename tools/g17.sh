#!/bin/bash
mkdir -p gpurun_out
timeout 400 python tools/plan_times.py x c4 > gpurun_out/plan_c4.txt 2>&1
timeout 400 python tools/tc2_trace.py paper_2408_01331_b200/_lib/variants/trace/libhnn_b200.so c4 > gpurun_out/trace_c4.txt 2>&1
echo done
