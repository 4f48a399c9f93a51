#!/bin/bash
# ncu evidence on the GPU box (B200_PROFILING.md): the bench launch list, DRAM traffic per launch
# including the write-back (tools/ncu_traffic.py), and one --set full capture of hdiff and vadv at
# 128x128x80.  Outputs under gpurun_out/<TAG>_*.
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=${TAG:-r02}
mkdir -p gpurun_out
# launch list of the bench command (cold-cache, serialised: compare shares, never absolute times)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --samples 100 --no-extras --no-cpu \
    --e2e-steps 1 --detail gpurun_out/${TAG}_ncu_bench_detail.json > gpurun_out/${TAG}_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/${TAG}_launches.log
for c in ${TRAFFIC_CONFIGS:-c2 c3}; do
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --cache-control none --clock-control none --replay-mode application --csv \
      --log-file gpurun_out/${TAG}_traffic_${c}.csv python tools/ncu_traffic.py run $c > gpurun_out/${TAG}_traffic_${c}.log 2>&1
  echo "traffic $c rc=$?" >> gpurun_out/${TAG}_traffic_${c}.log
done
for p in ${FULL_PROGRAMS:-hdiff vadv}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${p}_" -s 2 -c 1 \
      -o gpurun_out/${TAG}_full_${p} -f python tools/kernel_driver.py --program $p --domain 128 128 80 --reps 6 \
      > gpurun_out/${TAG}_full_${p}.log 2>&1
  echo "full $p rc=$?" >> gpurun_out/${TAG}_full_${p}.log
done
for f in gpurun_out/${TAG}_*.log; do tail -n 2 $f; done
