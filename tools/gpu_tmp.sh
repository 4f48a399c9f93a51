cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
: > gpurun_out/s3.jsonl
for rep in 1 2 3; do for v in s4 s3; do for dom in "128 128 80" "128 128 60"; do
  OEC_LIB_PATH=tune/$v.so timeout 300 python tools/kernel_bench.py --programs vadv --domain $dom --tag $v >> gpurun_out/s3.jsonl 2>&1
done; done; done
