#!/bin/bash
mkdir -p gpurun_out/p
O=gpurun_out/p
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for w in c5 c1 c2 c3; do timeout 300 python tools/plan_times.py x $w > $O/plan_$w.txt 2>&1; done
for w in c5 c1 c2; do timeout 600 python bench.py --workload $w --no-cpu > $O/bench_$w.json 2> $O/bench_$w.err; done
echo done
