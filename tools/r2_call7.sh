# round 2, call 7: A/B of the grad-W K-major B operands (MEFT_GW_KMAJOR) with per-GEMM ncu time / DRAM; COMPACT bench line
set -x
mkdir -p gpurun_out/c7
python bench.py --precision compact --skip-cpu-baseline > gpurun_out/c7/bench_compact.json 2> gpurun_out/c7/bench_compact.err
bash tools/ab_env.sh "X=0" "MEFT_GW_KMAJOR=1" > gpurun_out/c7/ab.log 2>&1
cp -r gpurun_out/ab gpurun_out/c7/ab_ncu
python bench.py --skip-cpu-baseline > gpurun_out/c7/bench_mixed.json 2> gpurun_out/c7/bench_mixed.err
echo done
