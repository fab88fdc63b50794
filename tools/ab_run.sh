# Developer A/B on the GPU box: step time (alternating) and per-GEMM time + DRAM bytes of each variant
mkdir -p gpurun_out/ab
for rep in 1 2; do for v in "$@"; do echo -n "$v "; MEFT_LIB=build/variants/$v.so python tools/profile_step.py 8 epilogue; done; done
for v in "$@"; do
  MEFT_LIB=build/variants/$v.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:k_gemm_bf16_pair --csv --log-file gpurun_out/ab/$v.csv python tools/profile_step.py 3 epilogue > /dev/null 2>&1
done
echo done
