#!/bin/bash
mkdir -p gpurun_out/w
O=gpurun_out/w
L=paper_2408_01331_b200/_lib
for i in 1 2; do
for v in base u8s1 u8s0 u4s1 fbs6 fbs8; do
  if [ $v = base ]; then lib=$L/libhnn_b200.so; else lib=$L/variants/$v/libhnn_b200.so; fi
  echo "== $v" >> $O/skinny_ab.txt
  timeout 300 python tools/plan_times.py $lib c3 2>&1 | grep -E 'simt16|skinny|sum' >> $O/skinny_ab.txt
done
done
echo done
