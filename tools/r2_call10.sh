# round 2, call 10: sharded (Python + C ABI) and drop-in tests after the owner-gather / activation_profile changes;
# the sharded step at world 1 through bench (both implementations)
set -x
mkdir -p gpurun_out/c10
python -m pytest tests/test_gpu_sharded.py tests/test_gpu_sharded_capi.py tests/test_gpu_peer.py tests/test_dropin.py -q -x > gpurun_out/c10/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c10/pytest.log
python bench.py --sharded --skip-cpu-baseline > gpurun_out/c10/bench_sharded_py.json 2> gpurun_out/c10/bench_sharded_py.err
python bench.py --sharded --sharded-impl capi --skip-cpu-baseline > gpurun_out/c10/bench_sharded_capi.json 2> gpurun_out/c10/bench_sharded_capi.err
python bench.py --skip-cpu-baseline > gpurun_out/c10/bench.json 2> gpurun_out/c10/bench.err
echo done
