#!/bin/bash
# full GPU pass: tests, smoke, bench (default), ncu launch list of the bench command, ncu --set full
# of the hot kernels.  Outputs in gpurun_out/ (scratch); summaries are copied into profiles/.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-r01}
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_$TAG.txt 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.txt
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"hdiff_|vadv_" -c 60 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 14 --warmup 3 --e2e-steps 0 --no-suite --no-cpu --sets 7 > gpurun_out/ncu_bench_$TAG.log 2>&1
for p in hdiff vadv; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"${p}_(tma|sp)" -s 2 -c 1 -o gpurun_out/prof_${p}_$TAG -f python tools/kernel_driver.py --program $p --reps 4 > gpurun_out/ncu_${p}_$TAG.log 2>&1
done
echo done
