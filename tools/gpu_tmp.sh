cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
bash tools/gpu_jit.sh
timeout 900 python bench.py --steps 3000 > gpurun_out/bench_jit3.json 2> gpurun_out/bench_jit3.err
