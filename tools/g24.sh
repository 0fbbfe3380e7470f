#!/bin/bash
mkdir -p gpurun_out/z
O=gpurun_out/z
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for w in c3 c2 c5 c1; do timeout 300 python tools/plan_times.py x $w > $O/plan_$w.txt 2>&1; done
echo done
