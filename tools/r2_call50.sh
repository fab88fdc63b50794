#!/bin/bash
# round 2, call 50: TMA L2 promotion of the operand maps (256 B default vs 128 B vs none), alternating 3 reps
set -x
mkdir -p gpurun_out/c50
for rep in 1 2 3; do
  echo "cfg default"; python tools/profile_step.py 12 epilogue mixed
  echo "cfg p128"; MEFT_LIB=build/variants/p128.so python tools/profile_step.py 12 epilogue mixed
  echo "cfg pnone"; MEFT_LIB=build/variants/pnone.so python tools/profile_step.py 12 epilogue mixed
done > gpurun_out/c50/steps.log 2>&1
echo done
