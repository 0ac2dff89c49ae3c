export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python scripts/fmm_profile_c5.py 1e-9 > gpurun_out/c5_e9.log 2>&1; cat gpurun_out/c5_e9.log
timeout 600 python scripts/fmm_profile_c5.py 1e-9 1000000 direct > gpurun_out/c5_e9_direct.log 2>&1; cat gpurun_out/c5_e9_direct.log
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,launch__grid_size,smsp__inst_executed.sum --clock-control none -k regex:"m2l_fused|first_kernel" --launch-skip 94 --csv --log-file gpurun_out/c5_m2l_ncu.csv python scripts/fmm_profile_c5.py 1e-9 > gpurun_out/c5_m2l_ncu.log 2>&1
echo rc=$?
# largest fused launch of the timed apply with source counters
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"m2l_fused" --launch-skip 92 -c 3 -f -o gpurun_out/c5_m2l_full python scripts/fmm_profile_c5.py 1e-9 > gpurun_out/c5_m2l_full.log 2>&1
echo rc=$?
