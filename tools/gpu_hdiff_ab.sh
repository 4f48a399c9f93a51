#!/bin/bash
# hdiff old/new (tune/liboec_{old,new}.so) at the sizes the tile tiers cover, f64 + f32, plus the
# GPU hdiff/pipeline tests with the new build.  TAG from the environment.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-hab}
OUT=gpurun_out/${TAG}.jsonl
: > $OUT
OEC_LIB_PATH=tune/liboec_new.so timeout 900 python -m pytest tests -m gpu -q -x -k "hdiff or pipeline or pipe or f32 or chain" 2>&1 | tail -2
for rep in 1 2; do for v in old new; do
  for dom in "128 128 80" "128 128 60" "256 256 60" "512 512 80" "1024 1024 80"; do
    for dt in f64 f32; do
      OEC_LIB_PATH=tune/liboec_$v.so timeout 300 python tools/kernel_bench.py --programs hdiff --domain $dom --dtype $dt --tag $v >> $OUT 2>&1
    done
  done
done; done
python - <<PY
import json, collections
a=collections.defaultdict(list)
for l in open("$OUT"):
    if l.startswith("{"):
        r=json.loads(l); a[(r["dtype"], tuple(r["domain"]), r["tag"])].append(r["us"])
for k,v in sorted(a.items()): print(k, min(v))
PY
