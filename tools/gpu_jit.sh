#!/bin/bash
# GPU check of the stencil-language JIT + the full GPU suite
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jit.py -x -q --timeout 300 > gpurun_out/pytest_jit.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_jit.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_all.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_all.txt
