# Developer A/B of runtime knobs: alternating step timings and per-GEMM ncu time / DRAM bytes per setting.
# usage: bash tools/ab_env.sh "ENV=a" "ENV=b" ...
mkdir -p gpurun_out/ab
for rep in 1 2 3; do for e in "$@"; do echo -n "$e "; env $e python tools/profile_step.py 8 epilogue; done; done
i=0
for e in "$@"; do
  env $e ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:k_gemm_bf16_pair --csv --log-file gpurun_out/ab/env$i.csv python tools/profile_step.py 3 epilogue > /dev/null 2>&1
  i=$((i+1))
done
echo done
