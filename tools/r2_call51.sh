#!/bin/bash
# round 2, call 51: persistent GEMM grid width under the power cap -- all 148 SMs vs 8 / 16 / 28 left idle
set -x
mkdir -p gpurun_out/c51
for rep in 1 2 3; do
  echo "cfg r0"; python tools/profile_step.py 12 epilogue mixed
  echo "cfg r8"; MEFT_GEMM_SM_RESERVE=8 python tools/profile_step.py 12 epilogue mixed
  echo "cfg r16"; MEFT_GEMM_SM_RESERVE=16 python tools/profile_step.py 12 epilogue mixed
  echo "cfg r28"; MEFT_GEMM_SM_RESERVE=28 python tools/profile_step.py 12 epilogue mixed
done > gpurun_out/c51/steps.log 2>&1
echo done
