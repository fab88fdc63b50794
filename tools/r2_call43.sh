#!/bin/bash
# round 2, call 43: small-FFN side-stream schedule (out / grad_h beside dA / grad-W): full suite, cfg1 timing, bench
set -x
mkdir -p gpurun_out/c43
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/c43/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c43/pytest.log
timeout 300 python tools/enqueue_bench.py cfg1 4 50 3 > gpurun_out/c43/enqueue_cfg1.jsonl 2>&1
MEFT_SMALL_STREAMS=0 timeout 300 python tools/enqueue_bench.py cfg1 4 50 3 > gpurun_out/c43/enqueue_cfg1_serial.jsonl 2>&1
timeout 600 python bench.py --workload cfg1 --skip-cpu-baseline > gpurun_out/c43/cfg1.json 2> gpurun_out/c43/cfg1.err
timeout 900 python bench.py > gpurun_out/c43/bench.json 2> gpurun_out/c43/bench.err
echo done
