# round 2, call 14: MIXED vs COMPACT (bf16 Adam moments) fused step, alternating, + per-GEMM ncu
set -x
mkdir -p gpurun_out/c14
for rep in 1 2 3; do for p in mixed compact; do python tools/profile_step.py 8 epilogue $p; done; done > gpurun_out/c14/steps.log 2>&1
for p in mixed compact; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:k_gemm_bf16_pair --csv --log-file gpurun_out/c14/$p.csv python tools/profile_step.py 3 epilogue $p > /dev/null 2>&1
done
echo done
