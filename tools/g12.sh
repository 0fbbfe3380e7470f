#!/bin/bash
# promotion width / register split variants of the pair GEMM: C3 per-launch times
mkdir -p gpurun_out
L=paper_2408_01331_b200/_lib/variants
for v in c16s0 c16s216 c32s216 c64s216 c32s200; do
  echo "== $v" >> gpurun_out/promo_ab.txt
  timeout 300 python tools/plan_times.py $L/$v/libhnn_b200.so c3 >> gpurun_out/promo_ab.txt 2>&1
done
for v in c16s0 c64s216; do
  echo "== $v c4" >> gpurun_out/promo_ab.txt
  timeout 300 python tools/plan_times.py $L/$v/libhnn_b200.so c4 2>&1 | grep -E 'tc2|sum' >> gpurun_out/promo_ab.txt
done
echo done
