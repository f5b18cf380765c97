#!/bin/bash
# setup-kernel change: parity tests, phase timings, ncu of the setup kernel
TAG=${1:-su}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_incremental.py -x -q --timeout 120 > gpurun_out/${TAG}_inc_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_inc_tests.log; tail -3 gpurun_out/${TAG}_inc_tests.log
for c in "resnet50 4096" "bert 4096" "vgg16 4096"; do timeout 90 python tools/time_inc.py $c; done > gpurun_out/${TAG}_time.jsonl 2> gpurun_out/${TAG}_time.err
cat gpurun_out/${TAG}_time.jsonl
timeout 300 ncu --set full --import-source on --clock-control none -k score_kernel_inc -s 2 -c 1 \
  -o gpurun_out/${TAG}_setup python tools/prof_score.py resnet50 4096 fp32 3 > gpurun_out/${TAG}_ncu_setup.log 2>&1
tail -2 gpurun_out/${TAG}_ncu_setup.log
