#!/bin/bash
# round 2, call 44: the grad-W GEMMs with an L2 evict_last hint on their small B operand (g / h, 64 MB) under the
# default raster (not tried before: only with N-fastest / 4-tile rasters), alternating with the default, 4 reps
set -x
mkdir -p gpurun_out/c44
for rep in 1 2 3 4; do
  python tools/profile_step.py 12 epilogue mixed
  MEFT_GEMM_GWB=0,0,2 MEFT_GEMM_GWA=0,0,2 python tools/profile_step.py 12 epilogue mixed
  MEFT_GEMM_GWB=0,1,2 MEFT_GEMM_GWA=0,1,2 python tools/profile_step.py 12 epilogue mixed
done > gpurun_out/c44/steps.log 2>&1
echo done
