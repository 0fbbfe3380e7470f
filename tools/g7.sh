#!/bin/bash
# full GPU suite, C4 split-K A/B, e2e loader threads, sanitizers, one-step ncu per workload (summaries only)
mkdir -p gpurun_out/san
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 400 python tools/plan_times.py x c4 > gpurun_out/plan_c4.txt 2>&1
HNN_CONV_SPLITK=0 timeout 400 python tools/plan_times.py x c4 > gpurun_out/plan_c4_nosplit.txt 2>&1
timeout 600 python bench.py --workload c4 --no-cpu --steps 10 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --no-cpu --loader-threads 14 > gpurun_out/bench_c3_t14.json 2> gpurun_out/bench_c3_t14.err
for prec in f32 bf16; do
  for tool in racecheck synccheck; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_step.py $prec > /tmp/san.log 2>&1
    echo "rc=$?" >> /tmp/san.log
    (head -60 /tmp/san.log; echo "[...]"; tail -40 /tmp/san.log) > gpurun_out/san/${tool}_${prec}.log
  done
done
for w in c3 c1 c2 c4 c5; do
  timeout 900 ncu --set full --profile-from-start off --clock-control none -o /tmp/step_$w -f python tools/profile_step.py $w > gpurun_out/ncu_step_$w.log 2>&1
  cp gpurun_out/plan_$w.json /tmp/ 2>/dev/null
  python tools/ncu_traffic.py /tmp/step_$w.ncu-rep gpurun_out/plan_$w.json $w > gpurun_out/traffic_$w.json 2> gpurun_out/traffic_$w.err
  python tools/ncu_summary.py --rep /tmp/step_$w.ncu-rep > gpurun_out/ncu_full_$w.txt 2>&1
done
du -sh gpurun_out
echo done
