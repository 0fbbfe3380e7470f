#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
HNN_BENCH_ONE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 20 --no-cpu > gpurun_out/bench_c3_n2.json 2> gpurun_out/bench_c3_n2.err
timeout 300 python tools/tc2_trace.py paper_2408_01331_b200/_lib/variants/trace/libhnn_b200.so c3 > gpurun_out/trace_c3.txt 2>&1
timeout 300 python tools/plan_times.py x c3 > gpurun_out/plan_c3.txt 2>&1
echo done
