#!/bin/bash
# K3 with one lane per candidate: parity tests, then the candidates-per-warp sweep (FO_K3_CPW)
TAG=${1:-k3l}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_incremental.py -x -q --timeout 120 > gpurun_out/${TAG}_inc_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_inc_tests.log; tail -5 gpurun_out/${TAG}_inc_tests.log
for c in 0 1 4 8 32; do
  if [ $c = 0 ]; then unset FO_K3_CPW; else export FO_K3_CPW=$c; fi
  echo "cpw=$c $(timeout 200 python tools/time_snap.py resnet50,bert,vgg16 4096 2>/dev/null | python -c 'import sys,json; [print(d["config"], d["inc_snap_ms"], d["inc_nosnap_ms"], d["k3_snap_ms"], d["k3_nosnap_ms"], d["bitexact_snap_vs_general"]) for d in map(json.loads, sys.stdin)]' | tr '\n' ' ')"
done | tee gpurun_out/${TAG}_sweep.txt
