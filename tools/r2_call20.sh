#!/bin/bash
# round 2, call 20: scale sweep refresh with the current build (one B200, T = 8192)
set -x
mkdir -p gpurun_out/c20
timeout 2400 python tools/scale_sweep.py 8192 4096:64:16 4096:64:128 16384:64:128 65536:256:16 65536:256:128 65536:256:512 \
    262144:1024:128 1048576:1024:16 1048576:1024:128 1048576:1024:512 > gpurun_out/c20/sweep.jsonl 2> gpurun_out/c20/sweep.err
echo done
