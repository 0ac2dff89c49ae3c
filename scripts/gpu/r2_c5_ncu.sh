export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"m2l_fused" --launch-skip 10 -c 1 -f -o gpurun_out/c5_m2l_full python scripts/fmm_profile_c5.py 1e-9 > gpurun_out/c5_m2l_full.log 2>&1
echo rc=$?
