#!/bin/bash
# One gpurun call: GPU tests, smoke, bench lines, ncu launch list + full capture of the top kernels.
# usage (from the repo root, on the box): bash tools/gpu_round.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
for w in c2 c5 c1; do
  timeout 600 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 600 python bench.py --workload c4 --no-cpu --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for w in c3 c2 c5; do timeout 300 python tools/plan_times.py x $w > gpurun_out/plan_$w.txt 2>&1; done
timeout 400 python tools/plan_times.py x c4 > gpurun_out/plan_c4.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
  python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'multi_tensor|gemm_tc2' -s 12 -c 6 \
  -o gpurun_out/prof_c3 python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_full_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'gemm_tc2|transpose_dy|im2col|wgrad_reduce' -s 20 -c 8 \
  -o gpurun_out/prof_c4 python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
  python bench.py --workload c4 --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch_c4.log 2>&1
echo done
