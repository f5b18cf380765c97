#!/bin/bash
# A/B of the successor prefetch in both loops (ring + shared-memory): parity, bench, latency phases
V=$PWD/paper_2209_12769_b200/_build/var/pf2/libdiscob200.so
FO_LIB_PATH=$V timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -1
FO_LIB_PATH=$V FO_TEAM=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -1
for r in 1 2; do for lib in default pf2; do
  if [ "$lib" = default ]; then unset FO_LIB_PATH; else export FO_LIB_PATH=$V; fi
  echo "== $lib"; timeout 300 python tools/time_latency_phases.py fp64 bert:1 bert:16 resnet50:1 vgg16:1 2>&1 | tail -5
done; done
unset FO_LIB_PATH
bash tools/gpu_lib_ab.sh pf2
