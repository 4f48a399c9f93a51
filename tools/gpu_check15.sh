#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu15.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu15.txt
timeout 600 python bench.py > gpurun_out/bench15.json 2> gpurun_out/bench15.err
