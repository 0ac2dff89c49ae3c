set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -p no:cacheprovider -m gpu tests/test_fmm_gpu.py tests/test_operators_gpu.py tests/test_sharding_gpu.py > gpurun_out/xw_tests.log 2>&1
echo "tests rc=$?"
tail -15 gpurun_out/xw_tests.log
timeout 900 python bench.py --no-cpu-baseline --no-extra > gpurun_out/bench_xw.log 2> gpurun_out/bench_xw.err
echo "bench rc=$?"
tail -3 gpurun_out/bench_xw.err
