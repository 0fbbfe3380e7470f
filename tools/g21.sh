#!/bin/bash
mkdir -p gpurun_out/x
O=gpurun_out/x
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 400 python tools/plan_times.py x c4 > $O/plan_c4.txt 2>&1
timeout 300 python tools/plan_times.py x c2 > $O/plan_c2.txt 2>&1
echo done
