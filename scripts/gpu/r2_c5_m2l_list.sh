export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for eps in 1e-9 1e-6; do
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread,dram__bytes_read.sum,dram__bytes_write.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"m2l|first_kernel|reduce_kernel" --launch-skip 0 -c 60 --csv --log-file gpurun_out/c5_m2l_list_$eps.csv python scripts/fmm_profile_c5.py $eps 1000000 direct > gpurun_out/c5_m2l_list_$eps.log 2>&1
echo rc=$?
done
