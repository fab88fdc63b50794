#!/bin/bash
# round 2, call 17: drop-in marshalling through page-locked staging (fused column walks, row-Adam, chunked uploads)
set -x
mkdir -p gpurun_out/c17
timeout 1200 python -m pytest tests/test_dropin.py tests/test_gpu_store.py -m gpu -x -q > gpurun_out/c17/dropin_tests.log 2>&1 || exit 1
timeout 1500 python tools/dropin_bench.py gpurun_out/c17/dropin_bench.jsonl > gpurun_out/c17/dropin_bench.log 2>&1
