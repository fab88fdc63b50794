#!/bin/bash
# round 2, call 53: 1-CTA kernel ring depth (4 default vs 3 vs 2) on the selection alone (cfg2 and M = 4,096) and cfg1
set -x
mkdir -p gpurun_out/c53
for rep in 1 2 3; do
  for v in default c1s3 c1s2; do
    if [ $v = default ]; then L=""; else L="MEFT_LIB=build/variants/$v.so"; fi
    echo "cfg $v"; env $L python tools/profile_select.py 20 certified 65536:256:128
    echo "cfg $v"; env $L python tools/profile_select.py 20 certified 4096:64:16
    echo "cfg $v"; env $L python tools/enqueue_bench.py cfg1 1 100 1 | tail -1
  done
done > gpurun_out/c53/steps.log 2>&1
echo done
