cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
OEC_BENCH_DEVICE=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 200 --warmup 3 --no-suite --no-cpu --e2e-steps 2 --dist-backend gloo > gpurun_out/bench_fused2.json 2> gpurun_out/bench_fused2.err
echo "exit $?" >> gpurun_out/bench_fused2.err
timeout 600 python bench.py --steps 600 --no-suite --no-cpu --e2e-steps 2 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
echo "exit $?" >> gpurun_out/bench_n1.err
