export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"m2l_fused|first_kernel" --launch-skip 34 --launch-count 4 -o gpurun_out/m2l_full -f python scripts/fmm_profile_c3.py > gpurun_out/m2l_full.log 2>&1
echo "rc=$?"
