#!/bin/bash
timeout 240 python -m pytest tests/test_gpu_incremental.py -x -q --timeout 60 2>&1 | tail -2
for sp in 0 1 0 1; do FO_INC_SPLIT=$sp timeout 120 python tools/time_inc.py resnet50 4096 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('split', $sp, d['mode1'])"; done
FO_INC_SPLIT=1 timeout 180 python bench.py --no-cpu-baseline --no-search | head -c 300; echo
