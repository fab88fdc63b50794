# round 2, call 3: probe + parity tests, GEMM L2/raster knob A/B, reference cost curve, 32-layer COMPACT stack
set -x
mkdir -p gpurun_out/c3
python -m pytest tests/test_gpu_tc_error_probe.py -q -s > gpurun_out/c3/probe.log 2>&1
python -m pytest tests/test_gpu_cfg2_parity.py tests/test_gpu_peer.py tests/test_gpu_compact.py -q -s > gpurun_out/c3/parity.log 2>&1
bash tools/ab_env.sh "X=0" "MEFT_GEMM_GWB=-1,0,2 MEFT_GEMM_GWA=-1,0,2" "MEFT_GEMM_GWB=-1,0,0 MEFT_GEMM_GWA=-1,0,0" \
   "MEFT_GEMM_GWB=4,0,2 MEFT_GEMM_GWA=4,0,2" "MEFT_GEMM_OUT=16,0,0 MEFT_GEMM_GH=16,0,0" \
   "MEFT_GEMM_OUT=4,0,0 MEFT_GEMM_GH=4,0,0" > gpurun_out/c3/ab.log 2>&1
cp -r gpurun_out/ab gpurun_out/c3/ab_ncu
python tools/stack_bench.py 32 16384 3 compact > gpurun_out/c3/stack32.json 2> gpurun_out/c3/stack32.err
python tools/ref_cost_curve.py 1 16 64 256 > gpurun_out/c3/refcurve.jsonl 2> gpurun_out/c3/refcurve.err
echo done
