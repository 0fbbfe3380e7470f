#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_workspace.py -q -x > gpurun_out/pytest_ws.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ws.log
timeout 300 python tools/adam_probe2.py 1024 2048 > gpurun_out/probe_chunk1.txt 2>&1
HNN_LIB_VARIANT=chunk2 timeout 300 python tools/adam_probe2.py 1024 2048 > gpurun_out/probe_chunk2.txt 2>&1
HNN_LIB_VARIANT=chunk2 timeout 300 python tools/plan_times.py x c3 > gpurun_out/plan_c3_chunk2.txt 2>&1
HNN_LIB_VARIANT=chunk2 timeout 600 python -m pytest tests/test_gpu_baseline_parity.py tests/test_gpu_parity.py -q -k "c3_width or single_step or trajectory" > gpurun_out/pytest_chunk2.log 2>&1
echo done
