# ncu evidence for the north-star per-kernel claims: HBM GB/s of gather / scatter / Adam (reference-API kernels,
# tools/profile_hbm.py) and tensor-pipe utilisation of the router and grouped key-scoring GEMMs (fused step).
mkdir -p gpurun_out/kern
python tools/profile_hbm.py 3 > gpurun_out/kern/hbm.txt 2>&1
ncu --set full --clock-control none -k regex:'k_gather2|k_stage_add|k_adam_mixed' --launch-skip 6 --launch-count 3 \
    -o gpurun_out/kern/hbm python tools/profile_hbm.py 3 > gpurun_out/kern/ncu_hbm.log 2>&1
ncu --set full --clock-control none -k regex:'^k_gemm_bf16$' --launch-skip 2 --launch-count 2 \
    -o gpurun_out/kern/select_gemm python tools/profile_step.py 2 > gpurun_out/kern/ncu_sel.log 2>&1
echo done
