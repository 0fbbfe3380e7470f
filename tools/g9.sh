#!/bin/bash
# Adam fast path: bit-exactness + timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py -x -q -m gpu -k "adam or optimizer or trajectory or single_step or c3_width or exact_div" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout 300 python tools/opt_variants.py paper_2408_01331_b200/_lib/libhnn_b200.so > gpurun_out/opt_fast.txt 2>&1
HNN_OPT_BULK=1 timeout 300 python tools/opt_variants.py paper_2408_01331_b200/_lib/libhnn_b200.so > gpurun_out/opt_fast_bulk.txt 2>&1
timeout 300 python tools/plan_times.py x c3 > gpurun_out/plan_c3.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo done
