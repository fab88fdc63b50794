#!/bin/bash
# round 2, call 15: enqueue-only layer step + CUDA graphs -- parity first, then the host-sync A/B
set -x
mkdir -p gpurun_out/c15
timeout 900 python -m pytest tests/test_gpu_enqueue_only.py -x -q -s > gpurun_out/c15/enqueue_tests.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q -k "layer or compact or select or store or sharded_capi or peer" > gpurun_out/c15/core_tests.log 2>&1
timeout 300 python tools/enqueue_bench.py cfg1 4 50 3 > gpurun_out/c15/enqueue_cfg1.jsonl 2>&1
timeout 600 python tools/enqueue_bench.py cfg2 4 5 3 > gpurun_out/c15/enqueue_cfg2.jsonl 2>&1
for m in sync enqueue graph; do
  timeout 900 python tools/stack_bench.py 32 16384 3 compact $m >> gpurun_out/c15/stack32.jsonl 2>&1
done
