#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu11.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu11.txt
: > gpurun_out/tune11.jsonl
python tools/kernel_bench.py --programs hdiff vadv --tag pdl >> gpurun_out/tune11.jsonl 2>&1
OEC_PDL=0 python tools/kernel_bench.py --programs hdiff vadv --tag nopdl >> gpurun_out/tune11.jsonl 2>&1
for f in tune/h_*.so; do OEC_LIB_PATH=$f python tools/kernel_bench.py --programs hdiff --tag $(basename $f .so) >> gpurun_out/tune11.jsonl 2>&1; done
python tools/kernel_bench.py --programs hdiff vadv --domain 1024 1024 80 --reps 5 --tag big >> gpurun_out/tune11.jsonl 2>&1
python tools/step_bench.py >> gpurun_out/tune11.jsonl 2>&1
