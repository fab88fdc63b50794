# Profiles committed under profiles/ (B200_PROFILING.md recipe): bench line, launch list of the same command,
# one --set full capture of a step's six FFN GEMMs (step 2 of tools/profile_step.py) and of the selection kernels.
set -x
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv \
    python bench.py --steps 2 --warmup 3 --skip-cpu-baseline > gpurun_out/prof/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gemm_bf16_pair --launch-skip 6 --launch-count 6 \
    -o gpurun_out/prof/gemm6 python tools/profile_step.py 2 epilogue > gpurun_out/prof/ncu_gemm6.log 2>&1
ncu --set full --clock-control none -k regex:'k_adam_mixed' --launch-skip 2 --launch-count 2 \
    -o gpurun_out/prof/adam_pass python tools/profile_step.py 2 pass > gpurun_out/prof/ncu_adam.log 2>&1
echo done
