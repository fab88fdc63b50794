#!/bin/bash
# round 2, call 60: bench.py with the default (synchronising) step vs the enqueue-only step (MEFT_HOST_SYNC=0), 3 reps
set -x
mkdir -p gpurun_out/c60
for rep in 1 2 3; do
  python bench.py --skip-cpu-baseline > gpurun_out/c60/sync_$rep.json 2>/dev/null
  MEFT_HOST_SYNC=0 python bench.py --skip-cpu-baseline > gpurun_out/c60/enq_$rep.json 2>/dev/null
done
echo done
