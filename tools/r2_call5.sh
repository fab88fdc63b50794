# round 2, call 5: full GPU suite, bench (+ phased cpu_baseline), drop-in API bench both ways, GEMM major sweep,
# launch list of the bench command
set -x
mkdir -p gpurun_out/c5
python -m pytest tests -m gpu -q -x > gpurun_out/c5/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c5/pytest.log
python bench.py > gpurun_out/c5/bench.json 2> gpurun_out/c5/bench.err; echo "rc=$?" >> gpurun_out/c5/bench.err
python tools/dropin_bench.py gpurun_out/c5/dropin_bench.jsonl > gpurun_out/c5/dropin_bench.log 2>&1
make -s -C tools gemm_check > gpurun_out/c5/gemm_build.log 2>&1 && tools/gemm_check perfmaj > gpurun_out/c5/perfmaj.txt 2>&1
python bench.py --steps 2 --warmup 3 --skip-cpu-baseline > gpurun_out/c5/b2.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5/launches.csv \
    python bench.py --steps 2 --warmup 3 --skip-cpu-baseline > gpurun_out/c5/ncu.log 2>&1
echo done
