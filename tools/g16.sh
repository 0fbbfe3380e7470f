#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/plan_times.py x c3 > gpurun_out/plan_c3.txt 2>&1
HNN_SKINNY_FUSED=0 timeout 300 python tools/plan_times.py x c3 > gpurun_out/plan_c3_nofuse.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo done
