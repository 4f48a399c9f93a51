cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu_all.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_all.txt
timeout 900 python bench.py --steps 3000 > gpurun_out/bench_jit4.json 2> gpurun_out/bench_jit4.err
