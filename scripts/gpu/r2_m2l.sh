set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -p no:cacheprovider -m gpu tests/test_fmm_gpu.py tests/test_dgemm_gpu.py > gpurun_out/m2l_tests.log 2>&1
echo "tests rc=$?"
tail -3 gpurun_out/m2l_tests.log
timeout 900 python scripts/m2l_modes.py > gpurun_out/m2l_modes.log 2>&1
echo "modes rc=$?"
grep -v staged gpurun_out/m2l_modes.log | grep -v "^fused"
grep "vs staged" gpurun_out/m2l_modes.log
bash scripts/gpu/r2_m2l_ncu.sh
bash scripts/gpu/r2_m2l_full.sh
