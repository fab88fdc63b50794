# round 2, call 6: drop-in + store + sharded tests, drop-in API bench (both libraries), compute-sanitizer memcheck
set -x
mkdir -p gpurun_out/c6
python -m pytest tests/test_dropin.py tests/test_gpu_store.py tests/test_gpu_sharded.py -q -x > gpurun_out/c6/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c6/pytest.log
python tools/dropin_bench.py gpurun_out/c6/dropin_bench.jsonl > gpurun_out/c6/dropin_bench.log 2>&1
python tools/sanitize_step.py > gpurun_out/c6/plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --log-file gpurun_out/c6/memcheck.txt python tools/sanitize_step.py > gpurun_out/c6/memcheck_run.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/c6/memcheck_run.log
echo done
