#!/bin/bash
# round 2, call 56: with the 4-stage ring, the gather choice (TMA default vs the gather kernel) and the act bitmask
# (default vs the bf16 act as the dA mask), alternating 3 reps
set -x
mkdir -p gpurun_out/c56
for rep in 1 2 3; do
  echo "cfg default"; python tools/profile_step.py 12 epilogue mixed
  echo "cfg gather_kernel"; MEFT_GATHER=kernel python tools/profile_step.py 12 epilogue mixed
  echo "cfg act_mask"; MEFT_ACT_BITS=0 python tools/profile_step.py 12 epilogue mixed
done > gpurun_out/c56/steps.log 2>&1
echo done
