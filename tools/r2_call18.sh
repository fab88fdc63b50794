#!/bin/bash
# round 2, call 18: full GPU suite + smoke, bench line, launch list of the bench command (after the enqueue-only /
# drop-in staging changes)
set -x
mkdir -p gpurun_out/c18
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/c18/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c18/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c18/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/c18/bench.json 2> gpurun_out/c18/bench.err; echo "rc=$?" >> gpurun_out/c18/bench.err
timeout 600 python bench.py --steps 2 --warmup 3 --skip-cpu-baseline > gpurun_out/c18/b2.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c18/launches.csv \
    python bench.py --steps 2 --warmup 3 --skip-cpu-baseline > gpurun_out/c18/ncu.log 2>&1
echo done
