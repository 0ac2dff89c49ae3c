export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
export BENCH_DIST_BACKEND=gloo BENCH_SHARE_GPU=1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_dist2.log 2> gpurun_out/bench_dist2.err
echo "dist2 rc=$?"
tail -2 gpurun_out/bench_dist2.log | cut -c1-1500
tail -5 gpurun_out/bench_dist2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/bench_dist2_ref.log 2> gpurun_out/bench_dist2_ref.err
echo "dist2 ref rc=$?"
tail -1 gpurun_out/bench_dist2_ref.log | cut -c1-300
