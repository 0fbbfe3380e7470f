#!/bin/bash
# GPU tests + sanitizer runs + per-workload one-step ncu captures (traffic / dram / tensor per kernel)
mkdir -p gpurun_out/san
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for prec in f32 bf16; do
  for tool in racecheck synccheck memcheck; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_step.py $prec > gpurun_out/san/${tool}_${prec}.log 2>&1
    echo "rc=$?" >> gpurun_out/san/${tool}_${prec}.log
  done
done
for w in c3 c1 c2 c4 c5; do
  timeout 900 ncu --set full --profile-from-start off --clock-control none -o gpurun_out/step_$w -f python tools/profile_step.py $w > gpurun_out/ncu_step_$w.log 2>&1
  python tools/ncu_traffic.py gpurun_out/step_$w.ncu-rep gpurun_out/plan_$w.json $w > gpurun_out/traffic_$w.json 2> gpurun_out/traffic_$w.err
  python tools/ncu_summary.py --rep gpurun_out/step_$w.ncu-rep > gpurun_out/ncu_full_$w.txt 2>&1
done
echo done
