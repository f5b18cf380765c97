#!/bin/bash
# bench launch list under ncu, the other configs, search, profiles of the final build
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-search > gpurun_out/r2_bench_under_ncu.log 2>&1
bash tools/gpu_r2_prof_inc.sh r2final > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k score_kernel_inc_mp -s 1 -c 1 -o gpurun_out/r2final_mp python tools/prof_score.py resnet50 4096 fp32 3 > /dev/null 2>&1
bash tools/gpu_r2_configs.sh > /dev/null 2>&1
bash tools/gpu_r2_search.sh
for f in r2_gpt2m_sweep r2_synth50k; do echo "== $f"; tail -c 400 gpurun_out/$f.json; echo; done
