#!/bin/bash
# round 2, call 19: selection alone across the sweep's geometries (time + launch lists)
set -x
mkdir -p gpurun_out/c19
for spec in 4096:64:16 65536:256:128 1048576:1024:128 1048576:1024:16; do
  timeout 300 python tools/profile_select.py 10 certified $spec >> gpurun_out/c19/select_times.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c19/launches_1m.csv \
    python tools/profile_select.py 3 certified 1048576:1024:128 > gpurun_out/c19/ncu1.log 2>&1
echo done
