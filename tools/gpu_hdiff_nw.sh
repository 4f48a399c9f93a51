cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for rep in 1 2; do for v in old n8 n8L n4L; do
  for dom in "128 128 80" "256 256 60" "512 512 80" "1024 1024 80"; do
    OEC_LIB_PATH=tune/liboec_$v.so timeout 300 python tools/kernel_bench.py --programs hdiff --domain $dom --tag $v >> gpurun_out/hn3.jsonl 2>&1
  done
  for dom in "128 128 80" "1024 1024 80"; do
    OEC_LIB_PATH=tune/liboec_$v.so timeout 300 python tools/kernel_bench.py --programs hdiff --domain $dom --dtype f32 --tag $v >> gpurun_out/hn3.jsonl 2>&1
  done
  for dom in "128 128 80" "512 512 80"; do OEC_LIB_PATH=tune/liboec_$v.so TAG=$v timeout 300 python tools/pipe_bench.py $dom >> gpurun_out/hn3.jsonl 2>&1; done
done; done
for v in n8L; do OEC_LIB_PATH=tune/liboec_$v.so timeout 900 python -m pytest tests -m gpu -q -x -k "hdiff or pipeline or pipe" 2>&1 | tail -2; done
python - <<'PY'
import json, collections
a=collections.defaultdict(list)
for l in open("gpurun_out/hn3.jsonl"):
    if not l.startswith("{"): continue
    r=json.loads(l)
    if "pipe_us" in r: a[("pipe", tuple(r["domain"]), r["tag"])].append((r["pipe_us"], r["hdiff_us"]))
    else: a[(r["program"]+r["dtype"], tuple(r["domain"]), r["tag"])].append(r["us"])
for k,v in sorted(a.items()): print(k, min(v), v)
PY
