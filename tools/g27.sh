#!/bin/bash
mkdir -p gpurun_out/v
O=gpurun_out/v
L=paper_2408_01331_b200/_lib
for i in 1 2; do
for v in base wg3; do
  if [ $v = base ]; then lib=$L/libhnn_b200.so; else lib=$L/variants/$v/libhnn_b200.so; fi
  for s in full 0/8 0/4 0/2; do
    echo "== $v $s" >> $O/wg3_ab.txt
    if [ $s = full ]; then timeout 300 python tools/plan_times.py $lib c3 2>&1 | grep -E 'tc2|sum' >> $O/wg3_ab.txt
    else timeout 300 python tools/plan_times.py $lib c3 $s 2>&1 | grep -E 'tc2|sum' >> $O/wg3_ab.txt; fi
  done
done
done
HNN_LIB_VARIANT=wg3 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py -x -q -m gpu > $O/wg3_pytest.txt 2>&1; echo "rc=$?" >> $O/wg3_pytest.txt
echo done
