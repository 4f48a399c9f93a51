#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu13.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu13.txt
timeout 600 python bench.py > gpurun_out/bench13.json 2> gpurun_out/bench13.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 \
  bench.py --gpus 1 --steps 3000 --warmup 5 --force-decomp > gpurun_out/bench13_decomp.json 2> gpurun_out/bench13_decomp.err
