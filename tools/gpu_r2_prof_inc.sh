#!/bin/bash
# timings of the sparse-candidate kernels + ncu --set full captures of the two incremental kernels
TAG=${1:-pinc}
mkdir -p gpurun_out
for c in "resnet50 4096" "bert 4096" "vgg16 4096"; do timeout 90 python tools/time_inc.py $c; done > gpurun_out/${TAG}_time.jsonl 2> gpurun_out/${TAG}_time.err
cat gpurun_out/${TAG}_time.jsonl
timeout 300 ncu --set full --import-source on --clock-control none -k regex:score_kernel_inc_k3 -s 2 -c 1 \
  -o gpurun_out/${TAG}_k3 python tools/prof_score.py resnet50 4096 fp32 3 > gpurun_out/${TAG}_ncu_k3.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k score_kernel_inc -s 2 -c 1 \
  -o gpurun_out/${TAG}_setup python tools/prof_score.py resnet50 4096 fp32 3 > gpurun_out/${TAG}_ncu_setup.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
  python tools/prof_score.py resnet50 4096 fp32 3 > gpurun_out/${TAG}_launches.csv 2>&1
tail -2 gpurun_out/${TAG}_ncu_k3.log gpurun_out/${TAG}_ncu_setup.log
grep -E "score_kernel|Kernel" gpurun_out/${TAG}_launches.csv | cut -c1-200 | head -20
