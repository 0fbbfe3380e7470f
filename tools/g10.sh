#!/bin/bash
# bulk optimizer variants (converged / early C3 state), per-thread kernel for reference
mkdir -p gpurun_out
L=paper_2408_01331_b200/_lib
for i in 1 2; do
timeout 300 python tools/opt_variants.py $L/libhnn_b200.so >> gpurun_out/opt_ab.txt 2>&1
HNN_OPT_BULK=1 timeout 300 python tools/opt_variants.py $L/libhnn_b200.so >> gpurun_out/opt_ab.txt 2>&1
for v in b32e4096s3 b16e4096s3 b16e2048s3c2 b8e1024s6c2; do
  HNN_OPT_BULK=1 timeout 300 python tools/opt_variants.py $L/variants/$v/libhnn_b200.so >> gpurun_out/opt_ab.txt 2>&1
done
done
echo done
