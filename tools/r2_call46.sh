#!/bin/bash
# round 2, call 46: pair-GEMM pipeline depth 6 (default) vs 4 vs 3, alternating 4 reps; per-GEMM ncu of 6 vs 4
set -x
mkdir -p gpurun_out/c46
for rep in 1 2 3 4; do
  python tools/profile_step.py 12 epilogue mixed
  MEFT_LIB=build/variants/st4.so python tools/profile_step.py 12 epilogue mixed
  MEFT_LIB=build/variants/st3.so python tools/profile_step.py 12 epilogue mixed
done > gpurun_out/c46/steps.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
ncu --metrics $M --clock-control none -k regex:k_gemm_bf16_pair --csv --log-file gpurun_out/c46/st6.csv python tools/profile_step.py 3 epilogue mixed > /dev/null 2>&1
MEFT_LIB=build/variants/st4.so ncu --metrics $M --clock-control none -k regex:k_gemm_bf16_pair --csv --log-file gpurun_out/c46/st4.csv python tools/profile_step.py 3 epilogue mixed > /dev/null 2>&1
echo done
