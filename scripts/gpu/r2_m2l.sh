export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -p no:cacheprovider -m gpu tests/test_fmm_gpu.py tests/test_dgemm_gpu.py tests/test_configs_gpu.py::test_config5_fmm_matches_reference_fmm > gpurun_out/m2l_tests.log 2>&1
echo "tests rc=$?"
tail -3 gpurun_out/m2l_tests.log
LB_FMM_DEBUG=1 timeout 900 python scripts/m2l_modes.py > gpurun_out/m2l_modes.log 2>&1
echo "modes rc=$?"
grep -v staged gpurun_out/m2l_modes.log | grep -v "^fused"
grep "vs staged" gpurun_out/m2l_modes.log
LB_FMM_DEBUG=1 python scripts/fmm_profile_c5.py 1e-9 2>&1 | grep "closed-form" 
