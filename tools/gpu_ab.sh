#!/bin/bash
# A/B timing of two liboec builds (tune/liboec_old.so vs tune/liboec_new.so) + vadv/hdiff parity
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
PROGS=${PROGS:-vadv}
OUT=gpurun_out/ab_${TAG:-x}.jsonl
: > $OUT
for rep in 1 2 3; do
  for v in old new; do
    for dom in "128 128 80" "1024 1024 80"; do
      OEC_LIB_PATH=tune/liboec_$v.so timeout 300 python tools/kernel_bench.py --programs $PROGS --domain $dom --tag $v >> $OUT 2>&1
    done
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/ab_parity_${TAG:-x}.txt 2>&1; echo "exit $?" >> gpurun_out/ab_parity_${TAG:-x}.txt
