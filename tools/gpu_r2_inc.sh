#!/bin/bash
# incremental delta kernel: parity vs the general kernel, then the bench with both modes
TAG=${1:-inc}
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_incremental.py -x -q --timeout 60 > gpurun_out/${TAG}_inc_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_inc_tests.log
tail -30 gpurun_out/${TAG}_inc_tests.log
timeout 180 python bench.py --no-cpu-baseline --no-search --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/%s_bench.json" % __import__("os").environ.get("TAG", "inc"))) if False else None
PY
head -c 400 gpurun_out/${TAG}_bench.json; echo; tail -3 gpurun_out/${TAG}_bench.err
