#!/bin/bash
# bulk Adam / colsum / skinny FWD / batched host gather: parity + A/B timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/plan_times.py x c3 > gpurun_out/plan_c3.txt 2>&1
HNN_OPT_BULK=0 timeout 300 python tools/plan_times.py x c3 > gpurun_out/plan_c3_nobulk.txt 2>&1
timeout 300 python tools/opt_variants.py paper_2408_01331_b200/_lib/libhnn_b200.so > gpurun_out/opt_bulk.txt 2>&1
HNN_OPT_BULK=0 timeout 300 python tools/opt_variants.py paper_2408_01331_b200/_lib/libhnn_b200.so > gpurun_out/opt_nobulk.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --workload c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo done
