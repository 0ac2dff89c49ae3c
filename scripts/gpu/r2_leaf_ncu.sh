set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python scripts/fmm_profile_c3.py 5e-8 400 direct > gpurun_out/c3_profile_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lattice_pot|leaf_kernel" --launch-skip 6 --launch-count 3 -f -o gpurun_out/c3_leaf_lattice python scripts/fmm_profile_c3.py 5e-8 400 direct > gpurun_out/c3_leaf_ncu.log 2>&1
echo "rc=$?"
ls -la gpurun_out/*.ncu-rep
