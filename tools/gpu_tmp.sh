cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_x.txt 2>&1; echo "exit $?" >> gpurun_out/smoke_x.txt
