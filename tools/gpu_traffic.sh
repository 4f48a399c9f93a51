#!/bin/bash
# DRAM traffic per launch incl. write-back for each configuration (tools/ncu_traffic.py)
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=${TAG:-r02}
mkdir -p gpurun_out
for c in ${TRAFFIC_CONFIGS:-c2 c3 c4 c5}; do
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --cache-control none --clock-control none --replay-mode application --csv \
      --log-file gpurun_out/${TAG}_traffic_${c}.csv python tools/ncu_traffic.py run $c > gpurun_out/${TAG}_traffic_${c}.log 2>&1
  echo "traffic $c rc=$?" >> gpurun_out/${TAG}_traffic_${c}.log
done
