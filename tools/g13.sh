#!/bin/bash
# 2-block chunks (grouped lo-first): accuracy vs float64 / oracle, C3 launch times, trace, parity subset
mkdir -p gpurun_out
L=paper_2408_01331_b200/_lib/variants
for v in default ck2; do
  if [ $v = default ]; then unset HNN_LIB_VARIANT; else export HNN_LIB_VARIANT=$v; fi
  echo "== $v" >> gpurun_out/ck_acc.txt
  timeout 600 python tools/adam_probe2.py 256 2048 >> gpurun_out/ck_acc.txt 2>&1
  echo "== $v" >> gpurun_out/ck_plan.txt
  timeout 300 python tools/plan_times.py x c3 >> gpurun_out/ck_plan.txt 2>&1
done
unset HNN_LIB_VARIANT
echo "== ck2c32" >> gpurun_out/ck_plan.txt
timeout 300 python tools/plan_times.py $L/ck2c32/libhnn_b200.so c3 >> gpurun_out/ck_plan.txt 2>&1
timeout 300 python tools/tc2_trace.py $L/ck2trace/libhnn_b200.so c3 > gpurun_out/ck_trace.txt 2>&1
HNN_LIB_VARIANT=ck2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py -q -m gpu > gpurun_out/ck_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/ck_pytest.txt
echo done
