cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 120 python tools/debug/jit_capture.py side > gpurun_out/dbg_side.txt 2>&1; echo "exit $?" >> gpurun_out/dbg_side.txt
timeout 120 python tools/debug/jit_capture.py cur > gpurun_out/dbg_cur.txt 2>&1; echo "exit $?" >> gpurun_out/dbg_cur.txt
