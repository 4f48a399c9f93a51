#!/bin/bash
# GPU check of the fused-exchange hdiff pipeline
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pipeline.py -m gpu -x -q > gpurun_out/pytest_pipe.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_pipe.txt
