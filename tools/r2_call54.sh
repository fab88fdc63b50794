#!/bin/bash
# round 2, call 54: evidence for the final (4-stage) build -- launch list of the bench command, then one
# --set full capture of the six FFN GEMMs of a steady-state step (the 4th step: 3 warm-ups skipped)
set -x
mkdir -p gpurun_out/c54
python bench.py --steps 2 --warmup 3 --skip-cpu-baseline > gpurun_out/c54/b2.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c54/launches.csv \
    python bench.py --steps 2 --warmup 3 --skip-cpu-baseline > gpurun_out/c54/ncu.log 2>&1
echo done
