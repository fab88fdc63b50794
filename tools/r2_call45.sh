#!/bin/bash
# round 2, call 45: pair-GEMM pipeline depth (6 default vs 5 vs 4 stages) and the Adam epilogue's evict-first
# streaming (default) vs plain loads / stores; alternating, 3 reps of profile_step 12
set -x
mkdir -p gpurun_out/c45
for rep in 1 2 3; do
  python tools/profile_step.py 12 epilogue mixed
  MEFT_LIB=build/variants/nostream.so python tools/profile_step.py 12 epilogue mixed
  MEFT_LIB=build/variants/st5.so python tools/profile_step.py 12 epilogue mixed
  MEFT_LIB=build/variants/st4.so python tools/profile_step.py 12 epilogue mixed
done > gpurun_out/c45/steps.log 2>&1
echo done
