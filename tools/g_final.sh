#!/bin/bash
# Round-end evidence: GPU suite, smoke, every workload's bench line, reference arm, per-launch
# breakdowns, ncu launch list (C3) and one-step ncu --set full per workload with DRAM traffic.
TAG=${1:-v6}
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 900 python -m pytest tests -q -m gpu > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $O/smoke_$TAG.log
timeout 600 python bench.py > $O/bench_c3_$TAG.json 2> $O/bench_c3_$TAG.err
for w in c5 c2 c1; do timeout 600 python bench.py --workload $w > $O/bench_${w}_$TAG.json 2> $O/bench_${w}_$TAG.err; done
timeout 600 python bench.py --workload c4 --no-cpu --steps 10 > $O/bench_c4_$TAG.json 2> $O/bench_c4_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err
HNN_BENCH_ONE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu > $O/bench_c3_2rank_onegpu_$TAG.json 2> $O/bench_c3_2rank_onegpu_$TAG.err
for w in c3 c5 c2 c1 c4; do timeout 400 python tools/plan_times.py x $w > $O/step_breakdown_${w}_$TAG.txt 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3_$TAG.csv \
  python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
for w in c3 c2 c5 c1; do
  timeout 900 ncu --set full --profile-from-start off --clock-control none -o /tmp/step_$w -f python tools/profile_step.py $w > /dev/null 2>&1
  python tools/ncu_traffic.py /tmp/step_$w.ncu-rep gpurun_out/plan_$w.json $w > $O/traffic_${w}_$TAG.json 2> $O/traffic_${w}_$TAG.err
  python tools/ncu_summary.py --rep /tmp/step_$w.ncu-rep > $O/ncu_step_${w}_$TAG.txt 2>&1
done
# C4 (140 launches): DRAM bytes + durations only (a --set full capture of every launch exceeds the timeout)
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --profile-from-start off \
  --clock-control none -o /tmp/step_c4 -f python tools/profile_step.py c4 > /dev/null 2>&1
python tools/ncu_traffic.py /tmp/step_c4.ncu-rep gpurun_out/plan_c4.json c4 > $O/traffic_c4_$TAG.json 2> $O/traffic_c4_$TAG.err
echo done
