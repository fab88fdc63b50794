# round 2, call 13: Adam-epilogue decomposition (A/B builds v0 shipped, v1 no HBM traffic, v3 no Adam math,
# v4 neither): live step timings alternating + per-GEMM ncu time / clock / DRAM / tensor activity
set -x
mkdir -p gpurun_out/c13
for rep in 1 2; do for v in e0 e1 e4 e5 e6; do echo -n "$v "; MEFT_LIB=build/variants/$v.so python tools/profile_step.py 8 epilogue; done; done > gpurun_out/c13/steps.log 2>&1
for v in e0 e1 e4 e5 e6; do
  MEFT_LIB=build/variants/$v.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum \
    --clock-control none -k regex:k_gemm_bf16_pair --csv --log-file gpurun_out/c13/$v.csv python tools/profile_step.py 3 epilogue > /dev/null 2>&1
done
echo done
