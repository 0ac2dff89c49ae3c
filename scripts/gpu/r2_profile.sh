set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python scripts/profile_step.py > gpurun_out/c3_launches.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none -k regex:"m2l_fused|gemm_cols|leaf_kernel|lattice_pot|csr_epi" -c 10 -o gpurun_out/c3_full python scripts/profile_step.py > gpurun_out/c3_full.log 2>&1
echo "full rc=$?"
timeout 900 python scripts/config5_sweep.py > gpurun_out/config5_sweep.jsonl 2> gpurun_out/config5_sweep.err
echo "sweep rc=$?"
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest -q -x -p no:cacheprovider tests/test_quadrature_gpu.py::test_corrections_match_reference tests/test_quadrature_gpu.py::test_near_map_bit_exact "tests/test_fmm_gpu.py::test_fmm_nonuniform_cloud_matches_reference" tests/test_fmm_gpu.py::test_device_tree_and_lists_equal_host tests/test_operators_gpu.py::test_apply_with_fmm_far_field tests/test_operators_gpu.py::test_gmres_matches_reference > gpurun_out/memcheck.log 2>&1
echo "memcheck rc=$?"
timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest -q -x -p no:cacheprovider "tests/test_quadrature_gpu.py::test_corrections_match_reference" tests/test_operators_gpu.py::test_gmres_matches_reference > gpurun_out/racecheck.log 2>&1
echo "racecheck rc=$?"
