#!/bin/bash
nvidia-smi -L
timeout 400 python -m pytest tests/test_gpu_multirank.py -q -x --timeout 300 > gpurun_out/mr_test.log 2>&1; tail -3 gpurun_out/mr_test.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2_bench_2gpu.json 2> gpurun_out/r2_bench_2gpu.err
head -c 700 gpurun_out/r2_bench_2gpu.json; echo; tail -3 gpurun_out/r2_bench_2gpu.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 5 --warmup 2 > gpurun_out/r2_bench_ref_2gpu.json 2>&1
head -c 300 gpurun_out/r2_bench_ref_2gpu.json
