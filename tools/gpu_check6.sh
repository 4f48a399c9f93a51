#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu6.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu6.txt
: > gpurun_out/tune6.jsonl
python tools/kernel_bench.py --programs hdiff vadv --tag default >> gpurun_out/tune6.jsonl 2>&1
for f in tune/v2_*.so; do OEC_LIB_PATH=$f timeout 120 python tools/kernel_bench.py --programs vadv --tag $(basename $f .so) >> gpurun_out/tune6.jsonl 2>&1; done
python tools/kernel_bench.py --programs hdiff vadv --domain 1024 1024 80 --reps 5 --tag big >> gpurun_out/tune6.jsonl 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"vadv_ws2" -s 2 -c 1 -o gpurun_out/prof6_vadv -f python tools/kernel_driver.py --program vadv --reps 4 > gpurun_out/ncu6_vadv.log 2>&1
echo done
