cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
: > gpurun_out/e2e_probe2.txt
for n in 1 2; do OEC_STAGE_SLABS=$n timeout 300 python tools/e2e_probe.py >> gpurun_out/e2e_probe2.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_jit.py -q --timeout 600 -k "host" > gpurun_out/pytest_host.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_host.txt
