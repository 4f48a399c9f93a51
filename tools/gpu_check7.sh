#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu7.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu7.txt
: > gpurun_out/tune7.jsonl
python tools/kernel_bench.py --programs hdiff vadv --tag default >> gpurun_out/tune7.jsonl 2>&1
OEC_LIB_PATH=tune/v_ws2.so python tools/kernel_bench.py --programs vadv --tag ws2 >> gpurun_out/tune7.jsonl 2>&1
python tools/kernel_bench.py --programs hdiff vadv --domain 1024 1024 80 --reps 5 --tag big >> gpurun_out/tune7.jsonl 2>&1
OEC_LIB_PATH=tune/vtrace.so python tools/vadv_trace.py > gpurun_out/vtrace4.txt 2>&1
echo done
