#!/bin/bash
# vadv A/B of tune/ builds + per-CTA traces (VA_TRACE builds).  VARIANTS, TRACES, TAG from the environment.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-vab}
for t in ${TRACES:-trace}; do
  OEC_LIB_PATH=tune/liboec_$t.so timeout 300 python tools/vadv_cta_trace.py --dtype ${DTYPE:-f64} > gpurun_out/${TAG}_trace_$t.txt 2>&1
  OEC_LIB_PATH=tune/liboec_$t.so timeout 300 python tools/vadv_cta_trace.py --dtype ${DTYPE:-f64} --domain 256 256 60 >> gpurun_out/${TAG}_trace_$t.txt 2>&1
done
VARIANTS="${VARIANTS:-old new}" PROGS=${PROGS:-vadv} DOMS="${DOMS:-128,128,80 256,256,60 1024,1024,80}" TAG=$TAG bash tools/gpu_ab.sh
python - <<'PY'
import json, os, collections
tag = os.environ.get("TAG", "vab")
rows = [json.loads(l) for l in open(f"gpurun_out/ab_{tag}.jsonl") if l.startswith("{")]
agg = collections.defaultdict(list)
for r in rows:
    agg[(r["tag"], r["program"], tuple(r.get("domain", ())))].append(r["us"])
for k, v in sorted(agg.items()):
    print(k, "us", sorted(v), "min", min(v))
PY
