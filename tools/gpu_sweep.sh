#!/bin/bash
# time several tuning builds (tune/<name>.so) of liboec on PROGS at 128^2 and 1024^2, 2 reps each
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
OUT=gpurun_out/sweep_${TAG:-x}.jsonl
: > $OUT
for rep in 1 2; do
  for v in $LIBS; do
    for dom in "128 128 80" "1024 1024 80"; do
      OEC_LIB_PATH=tune/$v.so timeout 300 python tools/kernel_bench.py --programs ${PROGS:-vadv} --domain $dom --tag $v >> $OUT 2>&1
    done
  done
done
