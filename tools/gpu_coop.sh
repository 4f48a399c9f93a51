#!/bin/bash
# A/B of tune/ builds (VARIANTS) for hdiff/vadv at 128^2 (f64, f32) + the L2-resident floor (--sets 1)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-coop}
OUT=gpurun_out/${TAG}.jsonl
: > $OUT
for rep in 1 2 3; do
  for v in ${VARIANTS:-old new}; do
    for dt in ${DTYPES:-f64 f32}; do
      OEC_LIB_PATH=tune/liboec_$v.so timeout 300 python tools/kernel_bench.py --programs ${PROGS:-vadv hdiff} --domain 128 128 80 --dtype $dt --tag $v >> $OUT 2>&1
    done
  done
done
[ -n "$NO_FLOOR" ] || for dt in f64 f32; do
  OEC_LIB_PATH=tune/liboec_old.so timeout 300 python tools/kernel_bench.py --programs vadv hdiff --domain 128 128 80 --dtype $dt --sets 1 --tag floor >> $OUT 2>&1
done
python - <<'PY'
import json, os, collections
tag = os.environ.get("TAG", "coop")
rows = [json.loads(l) for l in open(f"gpurun_out/{tag}.jsonl") if l.startswith("{")]
agg = collections.defaultdict(list)
for r in rows:
    agg[(r["tag"], r["program"], r["dtype"])].append(r["us"])
for k, v in sorted(agg.items()):
    print(k, "us", sorted(v), "min", min(v))
PY
