#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu14.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu14.txt
timeout 600 python bench.py > gpurun_out/bench14.json 2> gpurun_out/bench14.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 \
