#!/bin/bash
# compute-sanitizer racecheck + synccheck (+ memcheck) over every synchronising kernel
# (tools/sanitize.py); one log per (tool, case) under gpurun_out/sanitize/, summary at the end.
# Usage (on the GPU box): bash tools/sanitize.sh [case ...]
cd "$(dirname "$0")/.."
out=gpurun_out/sanitize
mkdir -p $out
cases=${@:-hdiff_tma hdiff_tma_large hdiff_pipe vadv_sp vadv_sp_pers vadv_sp_multi vadv_ragged jit_tiled}
for c in $cases; do
  for tool in racecheck synccheck memcheck; do
    extra=""
    [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --target-processes all \
      python tools/sanitize.py $c > $out/${tool}_$c.txt 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard|bit-identical' $out/${tool}_$c.txt | tr '\n' ' ')" >> $out/summary.txt
  done
done
cat $out/summary.txt
