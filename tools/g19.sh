#!/bin/bash
mkdir -p gpurun_out/x
O=gpurun_out/x
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for w in c3 c5 c1; do
  timeout 300 python tools/plan_times.py x $w > $O/plan_${w}_bulk.txt 2>&1
  HNN_SKINNY_FWD_BULK=0 timeout 300 python tools/plan_times.py x $w > $O/plan_${w}_warp.txt 2>&1
done
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --profile-from-start off --clock-control none -o /tmp/step_c4 -f python tools/profile_step.py c4 > $O/ncu_c4.log 2>&1
python tools/ncu_traffic.py /tmp/step_c4.ncu-rep gpurun_out/plan_c4.json c4 > $O/traffic_c4.json 2> $O/traffic_c4.err
echo done
