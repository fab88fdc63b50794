#!/bin/bash
# round 2, call 48: CTA-pair raster groups re-swept with the 4-stage ring (env knobs; alternating, 3 reps)
set -x
mkdir -p gpurun_out/c48
for rep in 1 2 3; do
  echo "cfg default"; python tools/profile_step.py 12 epilogue mixed
  echo "cfg AMN4"; MEFT_PAIR_GROUP_AMN=4 python tools/profile_step.py 12 epilogue mixed
  echo "cfg AMN16"; MEFT_PAIR_GROUP_AMN=16 python tools/profile_step.py 12 epilogue mixed
  echo "cfg BMN4"; MEFT_PAIR_GROUP_BMN=4 python tools/profile_step.py 12 epilogue mixed
  echo "cfg BMN16"; MEFT_PAIR_GROUP_BMN=16 python tools/profile_step.py 12 epilogue mixed
  echo "cfg KK8"; MEFT_PAIR_GROUP=8 MEFT_PAIR_GROUP_AMN=8 MEFT_PAIR_GROUP_BMN=8 python tools/profile_step.py 12 epilogue mixed
  echo "cfg KK32"; MEFT_PAIR_GROUP=32 MEFT_PAIR_GROUP_AMN=8 MEFT_PAIR_GROUP_BMN=8 python tools/profile_step.py 12 epilogue mixed
done > gpurun_out/c48/steps.log 2>&1
echo done
