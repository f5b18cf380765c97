#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_tensorcore.py -q -x --timeout 250 > gpurun_out/tc_test.log 2>&1; tail -3 gpurun_out/tc_test.log
cat gpurun_out/tensorcore_error.json
timeout 200 python tools/time_mp_arith.py resnet50 4096 > gpurun_out/tc_time_resnet50.json 2>&1; cat gpurun_out/tc_time_resnet50.json
timeout 200 python tools/time_mp_arith.py bert 4096 > gpurun_out/tc_time_bert.json 2>&1; cat gpurun_out/tc_time_bert.json
timeout 300 ncu --set full --import-source on --clock-control none -k score_kernel_inc_mp -s 1 -c 1 -o gpurun_out/r2_inc_mp python tools/prof_score.py resnet50 4096 fp32 3 > gpurun_out/r2_inc_mp_ncu.log 2>&1
tail -1 gpurun_out/r2_inc_mp_ncu.log
