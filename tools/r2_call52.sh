#!/bin/bash
# round 2, call 52: L2 hints with the 4-stage ring (env knobs; alternating, 3 reps): the streamed operand of each GEMM
# evict-first (out / grad_h: act / masked; z / dA: the keys / values table; grad-W: act^T / masked^T)
set -x
mkdir -p gpurun_out/c52
for rep in 1 2 3; do
  echo "cfg default"; python tools/profile_step.py 12 epilogue mixed
  echo "cfg outgh_a1"; MEFT_GEMM_OUT=0,1,0 MEFT_GEMM_GH=0,1,0 python tools/profile_step.py 12 epilogue mixed
  echo "cfg zda_b1"; MEFT_GEMM_Z=0,0,1 MEFT_GEMM_DA=0,0,1 python tools/profile_step.py 12 epilogue mixed
  echo "cfg gw_a1"; MEFT_GEMM_GWB=0,1,0 MEFT_GEMM_GWA=0,1,0 python tools/profile_step.py 12 epilogue mixed
  echo "cfg zda_a2"; MEFT_GEMM_Z=0,2,0 MEFT_GEMM_DA=0,2,0 python tools/profile_step.py 12 epilogue mixed
done > gpurun_out/c52/steps.log 2>&1
echo done
