# round 2, call 4: the C-ABI sharded step tests, then one full unsliced reference step (CPU, alone on the host)
set -x
mkdir -p gpurun_out/c4
python -m pytest tests/test_gpu_sharded_capi.py -q -s -x > gpurun_out/c4/capi.log 2>&1
python bench.py --impl reference --ref-full-step > gpurun_out/c4/ref_full.json 2> gpurun_out/c4/ref_full.err
echo done
