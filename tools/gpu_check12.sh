#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
: > gpurun_out/tune12.jsonl
for f in tune/h*.so; do OEC_LIB_PATH=$f python tools/kernel_bench.py --programs hdiff --tag $(basename $f .so) >> gpurun_out/tune12.jsonl 2>&1; OEC_LIB_PATH=$f python tools/kernel_bench.py --programs hdiff --domain 1024 1024 80 --reps 3 --tag $(basename $f .so)_big >> gpurun_out/tune12.jsonl 2>&1; done
