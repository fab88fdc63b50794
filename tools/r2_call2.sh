# round 2, call 2: cfg2 value parity, tcgen05 error probe, empty-union peer test, bench (phased CPU baseline), reference arm
set -x
mkdir -p gpurun_out/c2
python -m pytest tests/test_gpu_tc_error_probe.py tests/test_gpu_peer.py tests/test_gpu_cfg2_parity.py -x -q -s \
    > gpurun_out/c2/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/c2/pytest_new.log
python bench.py > gpurun_out/c2/bench.json 2> gpurun_out/c2/bench.err; echo "rc=$?" >> gpurun_out/c2/bench.err
python bench.py --impl reference > gpurun_out/c2/ref.json 2> gpurun_out/c2/ref.err; echo "rc=$?" >> gpurun_out/c2/ref.err
echo done
