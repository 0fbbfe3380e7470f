#!/bin/bash
# quick check of the split raw/lo rings + skinny/colsum changes: parity subset, A/B timings
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py -x -q -k "pair_tensor_core or trajectory or single_step or step_gradients or c3_width or optimizer_is_bit or host_fed or split_k or isolation or tf32" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
for v in default ring33 orig; do
  if [ $v = default ]; then unset HNN_LIB_VARIANT; else export HNN_LIB_VARIANT=$v; fi
  timeout 300 python tools/plan_times.py x c3 > gpurun_out/plan_c3_$v.txt 2>&1
done
unset HNN_LIB_VARIANT
timeout 300 python tools/plan_times.py x c5 > gpurun_out/plan_c5.txt 2>&1
timeout 300 python tools/plan_times.py x c1 > gpurun_out/plan_c1.txt 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo done
