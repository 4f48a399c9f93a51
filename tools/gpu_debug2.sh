#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out; out=gpurun_out/debug2.txt; : > $out
for args in "8 68 8 0 0" "8 68 8 2 0" "4 132 8 0 0" "4 132 8 2 0" "4 132 8 1 0" "4 128 8 0 0" "4 132 4 0 0" "4 68 8 0 0" "4 136 8 0 0" "4 132 8 -2 0" "8 68 8 -2 0" "4 132 8 2 8" "4 260 2 0 0" "4 196 8 0 0"; do
  timeout 20 tools/micro/tma_f32 $args >> $out 2>&1 || echo "rc $? for $args" >> $out
done
