#!/bin/bash
mkdir -p gpurun_out/san
for prec in ${SAN_PRECS:-f32 bf16}; do
  for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_step.py $prec > /tmp/san.log 2>&1
    echo "rc=$?" >> /tmp/san.log
    (head -40 /tmp/san.log; echo "[...]"; tail -25 /tmp/san.log) > gpurun_out/san/${tool}_${prec}_${SAN_TAG:-v13}.log
  done
done
echo done
