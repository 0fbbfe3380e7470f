#!/bin/bash
mkdir -p gpurun_out/x
O=gpurun_out/x
for w in c3 c5 c1 c2; do
  timeout 300 python tools/plan_times.py x $w > $O/plan_${w}_narrow.txt 2>&1
  HNN_TC_SKINNY_FWD=0 timeout 300 python tools/plan_times.py x $w > $O/plan_${w}_skinny.txt 2>&1
done
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --profile-from-start off --clock-control none -o /tmp/step_c4 -f python tools/profile_step.py c4 > /dev/null 2>&1
python tools/ncu_traffic.py /tmp/step_c4.ncu-rep gpurun_out/plan_c4.json c4 > $O/traffic_c4.json 2> $O/traffic_c4.err
echo done
