#!/bin/bash
# A/B: release-time loads addressed by one IMAD.WIDE each (wi)
R=$PWD/paper_2209_12769_b200/_build/var
FO_LIB_PATH=$R/wi/libdiscob200.so timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -1
FO_LIB_PATH=$R/wi/libdiscob200.so FO_TEAM=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -1
FO_LIB_PATH=$R/wi/libdiscob200.so FO_TEAM=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -1
FO_LIB_PATH=$R/wi/libdiscob200.so FO_SIM_SMEM=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -1
for r in 1; do for lib in default wi; do
  if [ "$lib" = default ]; then unset FO_LIB_PATH; else export FO_LIB_PATH=$R/$lib/libdiscob200.so; fi
  echo "== $lib"; timeout 300 python tools/time_latency_phases.py fp64 bert:1 bert:16 resnet50:1 vgg16:1 2>&1 | tail -4
done; done
unset FO_LIB_PATH
bash tools/gpu_lib_ab.sh wi
