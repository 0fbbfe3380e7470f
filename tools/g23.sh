#!/bin/bash
mkdir -p gpurun_out/y
O=gpurun_out/y
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for w in c5 c1 c3; do timeout 600 python bench.py --workload $w --no-cpu > $O/bench_$w.json 2> $O/bench_$w.err; done
HNN_HOSTFED_NATIVE=0 timeout 600 python bench.py --workload c5 --no-cpu > $O/bench_c5_py.json 2> $O/bench_c5_py.err
echo done
