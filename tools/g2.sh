#!/bin/bash
# GPU check: full gpu suite, C3 bench (N=1), the multi-rank bench on one GPU (gloo), reference arm,
# one-step ncu capture of C3 for the roofline traffic.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
HNN_BENCH_ONE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 20 --no-cpu > gpurun_out/bench_c3_n2.json 2> gpurun_out/bench_c3_n2.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --set full --profile-from-start off --clock-control none -o gpurun_out/step_c3 -f python tools/profile_step.py c3 > gpurun_out/ncu_step_c3.log 2>&1
python tools/ncu_traffic.py gpurun_out/step_c3.ncu-rep gpurun_out/plan_c3.json c3 > gpurun_out/traffic_c3.json 2> gpurun_out/traffic_c3.err
echo done
