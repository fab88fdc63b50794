# round 2, call 11: drop-in suites + API bench after threaded marshalling; ncu --set full of one step's six GEMMs
set -x
mkdir -p gpurun_out/c11
python -m pytest tests/test_dropin.py -q > gpurun_out/c11/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c11/pytest.log
python tools/dropin_bench.py gpurun_out/c11/dropin_bench.jsonl > gpurun_out/c11/dropin_bench.log 2>&1
python tools/profile_step.py 2 epilogue > gpurun_out/c11/ps.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemm_bf16_pair --launch-skip 6 --launch-count 6 \
    -o gpurun_out/c11/gemm6 python tools/profile_step.py 2 epilogue > gpurun_out/c11/ncu.log 2>&1
echo done
