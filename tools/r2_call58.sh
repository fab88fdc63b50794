#!/bin/bash
# round 2, call 58: e2e (meft_layer_step_host) with h uploaded before grad_out (default) vs both at once
set -x
mkdir -p gpurun_out/c58
for rep in 1 2 3; do
  python bench.py --skip-cpu-baseline > gpurun_out/c58/serial_$rep.json 2>/dev/null
  MEFT_H2D_SERIAL=0 python bench.py --skip-cpu-baseline > gpurun_out/c58/concurrent_$rep.json 2>/dev/null
done
echo done
