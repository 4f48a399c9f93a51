#!/bin/bash
# A/B timing of two liboec builds (tune/liboec_old.so vs tune/liboec_new.so) at several domains,
# interleaved 3 times.  PROGS, DOMS, TAG from the environment.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
PROGS=${PROGS:-vadv}
DOMS=${DOMS:-"128,128,80 1024,1024,80"}
OUT=gpurun_out/ab_${TAG:-x}.jsonl
: > $OUT
for rep in 1 2 3; do
  for v in ${VARIANTS:-old new}; do
    for dom in $DOMS; do
      OEC_LIB_PATH=tune/liboec_$v.so timeout 300 python tools/kernel_bench.py --programs $PROGS --domain ${dom//,/ } --dtype ${DTYPE:-f64} --tag $v >> $OUT 2>&1
    done
  done
done
