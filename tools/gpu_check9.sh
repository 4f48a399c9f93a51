#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu9.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu9.txt
: > gpurun_out/tune9.jsonl
python tools/kernel_bench.py --programs hdiff vadv --tag default >> gpurun_out/tune9.jsonl 2>&1
for f in tune/v*_*.so tune/h*_*.so; do [ -f $f ] && OEC_LIB_PATH=$f timeout 120 python tools/kernel_bench.py --programs hdiff vadv --tag $(basename $f .so) >> gpurun_out/tune9.jsonl 2>&1; done
python tools/kernel_bench.py --programs hdiff vadv --domain 1024 1024 80 --reps 5 --tag big >> gpurun_out/tune9.jsonl 2>&1
OEC_LIB_PATH=tune/vtrace.so python tools/vadv_trace.py > gpurun_out/vtrace9.txt 2>&1
echo done
