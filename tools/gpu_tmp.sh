cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
: > gpurun_out/f32_tiles.jsonl
for c in 0 2 3; do OEC_JIT_TILE_CFG=$c timeout 300 python tools/jit_tile_sweep.py --programs hdiff --dtype f32 >> gpurun_out/f32_tiles.jsonl 2>&1; done
timeout 300 python tools/jit_tile_sweep.py --programs hdiff --dtype f32 --variant 0 >> gpurun_out/f32_tiles.jsonl 2>&1
timeout 300 python tools/kernel_bench.py --programs hdiff --dtype f32 --tag builtin >> gpurun_out/f32_tiles.jsonl 2>&1
