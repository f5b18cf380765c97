#!/bin/bash
# event-loop fast-forward: parity tests, then the snapshot A/B and a bench line
TAG=${1:-snap}
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_incremental.py -x -q --timeout 120 > gpurun_out/${TAG}_inc_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_inc_tests.log
tail -15 gpurun_out/${TAG}_inc_tests.log
timeout 300 python tools/time_snap.py resnet50,bert,vgg16 4096 > gpurun_out/${TAG}_ab.jsonl 2> gpurun_out/${TAG}_ab.err
timeout 200 python tools/time_snap.py resnet50 4096 fp64 >> gpurun_out/${TAG}_ab.jsonl 2>> gpurun_out/${TAG}_ab.err
cat gpurun_out/${TAG}_ab.jsonl; tail -3 gpurun_out/${TAG}_ab.err
timeout 180 python bench.py --no-cpu-baseline --no-search --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
head -c 600 gpurun_out/${TAG}_bench.json; echo; tail -3 gpurun_out/${TAG}_bench.err
