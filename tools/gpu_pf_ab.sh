#!/bin/bash
# A/B of the successor prefetch at node start in the ring loop (FO_PREFETCH_SUCC variant lib)
V=$PWD/paper_2209_12769_b200/_build/var/pf/libdiscob200.so
FO_LIB_PATH=$V timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -1
FO_LIB_PATH=$V FO_TEAM=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -1
FO_LIB_PATH=$V FO_SIM_SMEM=0 timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -1
bash tools/gpu_lib_ab.sh pf
