#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out; out=gpurun_out/tune_f32.txt; : > $out
python tools/kernel_bench.py --programs vadv hdiff --dtype f32 --tag default >> $out 2>&1
for v in f_32_4_4 f_32_8_4 f_64_4_6 f_64_8_4 f_64_8_3 f_128_4_4 f_32_4_8 f_32_8_6; do
  OEC_LIB_PATH=tune/$v.so timeout 120 python tools/kernel_bench.py --programs vadv --dtype f32 --tag $v >> $out 2>&1
  OEC_LIB_PATH=tune/$v.so timeout 120 python tools/kernel_bench.py --programs vadv --dtype f32 --domain 1024 1024 80 --reps 5 --tag $v >> $out 2>&1
done
