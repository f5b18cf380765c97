#!/bin/bash
# full GPU suite + phase timings + one bench line
TAG=${1:-chk}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/${TAG}_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_pytest.log; tail -3 gpurun_out/${TAG}_pytest.log
for c in "resnet50 4096" "bert 4096" "vgg16 4096"; do timeout 90 python tools/time_inc.py $c; done > gpurun_out/${TAG}_time.jsonl 2> gpurun_out/${TAG}_time.err
cat gpurun_out/${TAG}_time.jsonl
timeout 180 python bench.py --no-cpu-baseline --no-search --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
head -c 400 gpurun_out/${TAG}_bench.json; echo
