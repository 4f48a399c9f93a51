#!/bin/bash
# first GPU pass: parity tests, smoke, short bench, ncu launch list + full captures
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.txt 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.txt
timeout 600 python bench.py --steps 3000 --warmup 10 --e2e-steps 5 --cpu-seconds 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 12 --warmup 3 --e2e-steps 0 --no-suite --no-cpu --sets 2 > gpurun_out/ncu_bench.log 2>&1
for p in hdiff vadv; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"${p}_" -s 2 -c 1 -o gpurun_out/prof_${p} -f python tools/kernel_driver.py --program $p --reps 4 > gpurun_out/ncu_${p}.log 2>&1
done
timeout 300 ncu --set full --clock-control none -k regex:hdiff_naive -s 2 -c 1 -o gpurun_out/prof_hdiff_naive -f python tools/kernel_driver.py --program hdiff --reps 4 --variant 2 > gpurun_out/ncu_hdiff_naive.log 2>&1
echo done
