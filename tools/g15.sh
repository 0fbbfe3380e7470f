#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "lenet or conv or c2 or direct or c4 or trajectory or isolation" > gpurun_out/pytest_conv.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_conv.log
timeout 300 python tools/plan_times.py x c2 > gpurun_out/plan_c2.txt 2>&1
ncu --set full --profile-from-start off --clock-control none -k regex:"conv_direct" -o gpurun_out/cd2_c2 -f python tools/profile_step.py c2 > gpurun_out/cd2.log 2>&1
echo done
