#!/bin/bash
# BERT 256 seeds on 4 GPUs: exchange once vs every round at several lags
TAG=${1:-xv}
mkdir -p gpurun_out
: > gpurun_out/${TAG}_variants.jsonl
for v in "end 0" "round 8" "round 1" "round 32" "round 8" "end 0"; do
  set -- $v
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 \
    tools/bench_search.py --config bert --seeds 64 --oracle-seeds 0 --exchange $1 --lag $2 2>/dev/null | grep '"metric"' >> gpurun_out/${TAG}_variants.jsonl
done
python -c "
import json
for l in open('gpurun_out/${TAG}_variants.jsonl'):
    d=json.loads(l); print(d['exchange'], d['lag'], d['exchanges'], round(d['wall_s'],3), d['best_cost_us'], d['best_seed'], round(d['rank0_expand_ms']), round(d['rank0_device_ms']))
"
