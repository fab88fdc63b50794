# A/B of the fused step's Adam placement: timing, then serialized launch lists (tools/profile_step.py)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests.log
for i in 1 2; do python tools/profile_step.py 8 epilogue; python tools/profile_step.py 8 pass; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_epi.csv python tools/profile_step.py 3 epilogue > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gemm_bf16_pair --launch-skip 10 --launch-count 2 -o gpurun_out/adam_epi python tools/profile_step.py 3 epilogue > gpurun_out/ncu_full.log 2>&1
echo done
