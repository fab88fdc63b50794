set -x
mkdir -p gpurun_out/c1
nvidia-smi > gpurun_out/c1/smi.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/c1/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c1/pytest.log
python bench.py --skip-cpu-baseline > gpurun_out/c1/bench.json 2> gpurun_out/c1/bench.err
python tools/profile_step.py 2 epilogue > gpurun_out/c1/ps.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemm_bf16_pair --launch-skip 10 --launch-count 2 \
    -o gpurun_out/c1/adamgemm python tools/profile_step.py 2 epilogue > gpurun_out/c1/ncu.log 2>&1
nproc > gpurun_out/c1/nproc.txt; lscpu > gpurun_out/c1/lscpu.txt; free -g >> gpurun_out/c1/lscpu.txt
echo done
