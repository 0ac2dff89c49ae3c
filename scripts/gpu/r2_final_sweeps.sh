export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python scripts/shard_projection_r2.py config3 400 > gpurun_out/shard_projection_c3.jsonl 2> gpurun_out/shard_projection_c3.err
echo "c3 rc=$?"
timeout 2400 python scripts/shard_projection_r2.py config4 400 > gpurun_out/shard_projection_c4.jsonl 2> gpurun_out/shard_projection_c4.err
echo "c4 rc=$?"
timeout 1500 python scripts/config5_sweep.py > gpurun_out/config5_sweep.jsonl 2> gpurun_out/config5_sweep.err
echo "sweep rc=$?"
tail -3 gpurun_out/config5_sweep.err
