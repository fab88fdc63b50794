#!/bin/bash
# round 2, call 49: bench.py itself, 4-stage (default build) vs 6-stage ring (variant), alternating 3 reps
set -x
mkdir -p gpurun_out/c49
for rep in 1 2 3; do
  python bench.py --skip-cpu-baseline > gpurun_out/c49/st4_$rep.json 2>/dev/null
  MEFT_LIB=build/variants/st6.so python bench.py --skip-cpu-baseline > gpurun_out/c49/st6_$rep.json 2>/dev/null
done
echo done
