# round 2, call 9: Adam-epilogue experiments (A/B builds, step timings + per-GEMM ncu), then the guard-zone suite
set -x
mkdir -p gpurun_out/c9
bash tools/ab_run.sh v0 v1 v2 > gpurun_out/c9/ab_adam.log 2>&1
cp -r gpurun_out/ab gpurun_out/c9/ab_ncu
for rep in 1 2; do echo -n "pass "; MEFT_ADAM_EPILOGUE=0 python tools/profile_step.py 8 pass; echo -n "epi "; python tools/profile_step.py 8 epilogue; done > gpurun_out/c9/pass_vs_epi.log 2>&1
MEFT_GUARD_ZONES=1 python -m pytest tests -m gpu -q > gpurun_out/c9/guard_suite.log 2>&1; echo "rc=$?" >> gpurun_out/c9/guard_suite.log
echo done
