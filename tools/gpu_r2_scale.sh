#!/bin/bash
for n in 2 4; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --steps 20 --warmup 5 2>/dev/null | grep "^{" > gpurun_out/r2_bench_${n}gpu.json
python -c "import json; d=json.load(open('gpurun_out/r2_bench_${n}gpu.json')); print($n, d['value'], d['e2e']['value'], d['ms_per_step'])"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29520 tools/bench_configs.py synth50k 2>/dev/null | grep "^{" > gpurun_out/r2_synth50k_4gpu.json; tail -c 300 gpurun_out/r2_synth50k_4gpu.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 tools/bench_search.py --config bert --seeds 64 --oracle-seeds 0 2>/dev/null | grep "^{" > gpurun_out/r2_search_bert_64_4gpu.json; tail -c 400 gpurun_out/r2_search_bert_64_4gpu.json
