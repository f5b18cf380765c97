#!/bin/bash
# timings of the sparse-candidate kernels + one ncu --set full capture of the incremental kernel
TAG=${1:-pinc}
mkdir -p gpurun_out
for c in "resnet50 4096" "bert 4096" "vgg16 4096"; do timeout 300 python tools/time_inc.py $c; done > gpurun_out/${TAG}_time.jsonl 2> gpurun_out/${TAG}_time.err
cat gpurun_out/${TAG}_time.jsonl
timeout 600 ncu --set full --import-source on --clock-control none -k regex:score_kernel_inc -s 2 -c 1 \
  -o gpurun_out/${TAG}_inc python tools/prof_score.py resnet50 4096 fp32 3 > gpurun_out/${TAG}_ncu.log 2>&1
tail -3 gpurun_out/${TAG}_ncu.log
