export PYTHONUNBUFFERED=1
for mb in 256 1024 4096 16384; do
  echo "cap $mb"; LB_M2L_PART_MB=$mb python scripts/fmm_profile_c5.py 1e-9 2>&1 | grep -o "'m2l': [0-9.]*"
done
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"m2l_fused|first_kernel|reduce_kernel" --launch-skip 58 --csv --log-file gpurun_out/c5_m2l_ncu.csv python scripts/fmm_profile_c5.py 1e-9 > gpurun_out/c5_m2l_ncu.log 2>&1
