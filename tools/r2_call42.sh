#!/bin/bash
# round 2, call 42: full GPU suite + smoke + bench after the small-Adam-on-pairs / C-ABI sharded peer + overlap /
# drop-in staging changes
set -x
mkdir -p gpurun_out/c42
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/c42/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c42/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c42/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/c42/bench.json 2> gpurun_out/c42/bench.err; echo "rc=$?" >> gpurun_out/c42/bench.err
echo done
