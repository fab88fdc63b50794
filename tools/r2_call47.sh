#!/bin/bash
# round 2, call 47: 4-stage pair GEMM as the default -- full suite, bench (cfg2), cfg4, cfg3 stack
set -x
mkdir -p gpurun_out/c47
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/c47/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c47/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c47/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/c47/bench.json 2> gpurun_out/c47/bench.err
timeout 900 python bench.py --workload cfg4 --skip-cpu-baseline > gpurun_out/c47/cfg4.json 2> gpurun_out/c47/cfg4.err
timeout 900 python tools/stack_bench.py 32 16384 3 compact graph > gpurun_out/c47/stack32_graph.json 2>&1
echo done
