#!/bin/bash
# BERT 256 seeds on 4 GPUs: exchange once vs every round, native NCCL exchange (fo_xchg) vs the
# torch.distributed one on a Python thread (FO_XCHG_PY=1), interleaved and repeated
TAG=${1:-xv6}
mkdir -p gpurun_out
: > gpurun_out/${TAG}_variants.jsonl
for rep in 1 2; do
for v in "end 0 0" "round 8 0" "round 8 1" "round 64 0"; do
  set -- $v
  if [ $3 = 1 ]; then export FO_XCHG_PY=1; else unset FO_XCHG_PY; fi
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 \
    tools/bench_search.py --config bert --seeds 64 --oracle-seeds 0 --exchange $1 --lag $2 2>/dev/null | grep '"metric"' | sed "s/}\$/, \"py\": $3}/" >> gpurun_out/${TAG}_variants.jsonl
done
done
python -c "
import json
for l in open('gpurun_out/${TAG}_variants.jsonl'):
    d=json.loads(l); print(d['exchange'], d['lag'], 'py' if d['py'] else 'native', d['exchanges'], round(d['wall_s'],3), d['best_seed'], round(d['rank0_expand_ms']), round(d['rank0_device_ms']))
"
