set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err
echo "bench ref rc=$?"
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python scripts/profile_step.py > gpurun_out/c3_launches.log 2>&1
echo "launches rc=$?"
