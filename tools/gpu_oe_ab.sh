#!/bin/bash
# A/B: opaque indegree/successor pointers in the linear-buffer event loop (large graphs, timelines)
V=$PWD/paper_2209_12769_b200/_build/var/oe/libdiscob200.so
FO_LIB_PATH=$V timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -1
FO_LIB_PATH=$V FO_SIM_SMEM=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -1
for r in 1 2; do for lib in default oe; do
  if [ "$lib" = default ]; then unset FO_LIB_PATH; else export FO_LIB_PATH=$V; fi
  echo "== $lib"; timeout 600 python tools/bench_configs.py synth50k --batch 8192 2>/dev/null | tail -1 | cut -c1-330
done; done
unset FO_LIB_PATH
bash tools/gpu_lib_ab.sh oe 2>&1 | head -8
