#!/bin/bash
mkdir -p gpurun_out/r
O=gpurun_out/r
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for s in full 0/8 0/4 0/2; do
  echo "== $s" >> $O/ring.txt
  if [ $s = full ]; then timeout 300 python tools/plan_times.py x c3 2>&1 | grep -E 'tc2|sum' >> $O/ring.txt
  else timeout 300 python tools/plan_times.py x c3 $s 2>&1 | grep -E 'tc2|sum' >> $O/ring.txt; fi
done
for w in c5 c1 c2; do echo "== $w" >> $O/ring.txt; timeout 300 python tools/plan_times.py x $w 2>&1 | grep -E 'tc2|sum' >> $O/ring.txt; done
echo done
