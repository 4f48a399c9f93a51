cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_final.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_final.txt
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_final.txt 2>&1; echo "exit $?" >> gpurun_out/smoke_final.txt
