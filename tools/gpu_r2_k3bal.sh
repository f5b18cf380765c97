#!/bin/bash
# K3 with a candidate counter: event-loop warps per SM sweep (FO_K3_BLOCKS_PER_SM), snapshots on/off
TAG=${1:-k3b}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_incremental.py -x -q --timeout 120 > gpurun_out/${TAG}_inc_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_inc_tests.log; tail -3 gpurun_out/${TAG}_inc_tests.log
for b in 0 7 6 5 4 3; do
  if [ $b = 0 ]; then unset FO_K3_BLOCKS_PER_SM; else export FO_K3_BLOCKS_PER_SM=$b; fi
  echo "bps=$b $(timeout 200 python tools/time_snap.py resnet50,bert 4096 2>/dev/null | python -c 'import sys,json; [print(d["config"], d["inc_snap_ms"], d["inc_nosnap_ms"], d["k3_snap_ms"], d["k3_nosnap_ms"], d["bitexact_snap_vs_general"]) for d in map(json.loads, sys.stdin)]' | tr '\n' ' ')"
done | tee gpurun_out/${TAG}_sweep.txt
