cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
: > gpurun_out/vpersist2.jsonl
for dom in "128 128 80" "256 256 60" "384 384 80" "512 512 80" "1024 1024 80"; do
  timeout 300 python tools/kernel_bench.py --programs vadv --domain $dom --tag tmpl2 >> gpurun_out/vpersist2.jsonl 2>&1
done
for dom in "256 256 60" "1024 1024 80"; do
  timeout 300 python tools/kernel_bench.py --programs vadv --dtype f32 --domain $dom --tag tmpl2_32 >> gpurun_out/vpersist2.jsonl 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f32.py -q --timeout 600 -x -k vadv > gpurun_out/pytest_v.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_v.txt
