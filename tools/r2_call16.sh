#!/bin/bash
# round 2, call 16: enqueue-only step with the estimated gather choice (kernel gather padded for sparse unions)
set -x
mkdir -p gpurun_out/c16
timeout 900 python -m pytest tests/test_gpu_enqueue_only.py -x -q -s > gpurun_out/c16/enqueue_tests.log 2>&1 || exit 1
timeout 300 python tools/enqueue_bench.py cfg1 4 50 3 > gpurun_out/c16/enqueue_cfg1.jsonl 2>&1
timeout 600 python tools/enqueue_bench.py cfg2 4 5 3 > gpurun_out/c16/enqueue_cfg2.jsonl 2>&1
