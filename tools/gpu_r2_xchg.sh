#!/bin/bash
# lagged per-round exchange: 2-rank GPU tests, then BERT 256 seeds on 4 GPUs, exchange every round vs once
TAG=${1:-xc}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multirank.py -x -q --timeout 300 > gpurun_out/${TAG}_multirank.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_multirank.log; tail -3 gpurun_out/${TAG}_multirank.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 \
  tools/bench_search.py --config bert --seeds 64 --oracle-seeds 0 > gpurun_out/${TAG}_bert256_4gpu.json 2> gpurun_out/${TAG}_bert256_4gpu.err
grep -v NCCL gpurun_out/${TAG}_bert256_4gpu.json | tail -1 | head -c 700; echo
tail -3 gpurun_out/${TAG}_bert256_4gpu.err
