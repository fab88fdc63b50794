# round 2, call 8: the guard-zone tests, then the whole -m gpu suite with MEFT_GUARD_ZONES=1
set -x
mkdir -p gpurun_out/c8
python -m pytest tests/test_gpu_guard.py -q > gpurun_out/c8/guard_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c8/guard_tests.log
MEFT_GUARD_ZONES=1 python -m pytest tests -m gpu -q > gpurun_out/c8/guard_suite.log 2>&1; echo "rc=$?" >> gpurun_out/c8/guard_suite.log
echo done
