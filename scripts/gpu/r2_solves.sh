export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python scripts/config3_solve.py 5e-8 400 3 > gpurun_out/config3_solve.json 2> gpurun_out/config3_solve.err
echo "c3 rc=$?"; tail -2 gpurun_out/config3_solve.err
timeout 1500 python scripts/config3_solve.py 1e-9 400 4 > gpurun_out/config4_solve.json 2> gpurun_out/config4_solve.err
echo "c4 rc=$?"; tail -2 gpurun_out/config4_solve.err
