#!/bin/bash
# K3 (event loop) instruction / cycle metrics with and without the parent snapshots
TAG=${1:-k3m}
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_elapsed.max,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
for v in snap nosnap; do
  if [ $v = nosnap ]; then export FO_INC_NO_SNAP=1; else unset FO_INC_NO_SNAP; fi
  timeout 300 ncu --metrics $M --clock-control none -k regex:score_kernel_inc_k3 -s 2 -c 1 --csv \
    python tools/prof_score.py resnet50 4096 fp32 3 > gpurun_out/${TAG}_${v}.csv 2>&1
  grep -E "inst_executed|cycles|duration|issue_active|warps_active" gpurun_out/${TAG}_${v}.csv | awk -F'","' '{print "'$v'", $(NF-2), $NF}'
done
