export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -x -p no:cacheprovider -m gpu tests/test_operators_gpu.py tests/test_sharding_gpu.py tests/test_sharding_dist_gpu.py tests/test_configs_gpu.py > gpurun_out/quick_tests.log 2>&1
echo "tests rc=$?"
tail -5 gpurun_out/quick_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_quick.log 2> gpurun_out/bench_quick.err
echo "bench rc=$?"
tail -3 gpurun_out/bench_quick.err
