#!/bin/bash
# One validation pass on the GPU box: GPU tests, smoke, the default bench (+ reference arm) and the
# multi-GPU configurations at N=1.  Outputs under gpurun_out/<TAG>_*.
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=${TAG:-r02}
mkdir -p gpurun_out
if [ -z "$NO_TESTS" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.txt
fi
timeout 900 python bench.py --detail gpurun_out/${TAG}_bench_detail.json > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_ref.json 2>&1
for c in ${CONFIGS:-c3 c4 c5}; do
  timeout 900 python bench.py --config $c --no-extras --no-cpu --detail gpurun_out/${TAG}_bench_${c}_detail.json > gpurun_out/${TAG}_bench_${c}.json 2> gpurun_out/${TAG}_bench_${c}.err; echo "rc=$?" >> gpurun_out/${TAG}_bench_${c}.err
done
tail -3 gpurun_out/${TAG}_pytest_gpu.txt 2>/dev/null; tail -2 gpurun_out/${TAG}_smoke.txt 2>/dev/null
tail -c 2500 gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
for c in ${CONFIGS:-c3 c4 c5}; do tail -c 1500 gpurun_out/${TAG}_bench_${c}.json; tail -2 gpurun_out/${TAG}_bench_${c}.err; done
