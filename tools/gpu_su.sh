#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_su.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_su.txt
: > gpurun_out/su.jsonl
P="uvbke p_grad_c nh_p_grad fvtp2d_qi fvtp2d_qj fvtp2d_flux fastwaves"
python tools/kernel_bench.py --programs $P --tag default >> gpurun_out/su.jsonl 2>&1
for f in tune/su_*.so; do OEC_LIB_PATH=$f python tools/kernel_bench.py --programs $P --tag $(basename $f .so) >> gpurun_out/su.jsonl 2>&1; done
