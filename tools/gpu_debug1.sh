#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
out=gpurun_out/debug1.txt; : > $out
for v in 0 1 2 3; do for p in hdiff uvbke; do
  timeout 60 python tools/debug/f32_probe.py $p $v f32 >> $out 2>&1 || echo "FAIL $p $v" >> $out
done; done
timeout 60 python tools/debug/f32_probe.py vadv 0 f32 >> $out 2>&1 || echo "FAIL vadv 0" >> $out
timeout 120 compute-sanitizer --tool memcheck python tools/debug/f32_probe.py hdiff 0 f32 > gpurun_out/debug1_san.txt 2>&1
