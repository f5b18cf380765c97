#!/bin/bash
timeout 300 python tools/bench_search.py --config vgg16 --seeds 1 > gpurun_out/r2_search_vgg16.json 2>&1
timeout 600 python tools/bench_search.py --config bert --seeds 1 > gpurun_out/r2_search_bert_1.json 2>&1
timeout 600 python tools/bench_search.py --config bert --seeds 16 --oracle-seeds 0 > gpurun_out/r2_search_bert_16.json 2>&1
timeout 600 python tools/bench_search.py --config bert --seeds 64 --oracle-seeds 0 > gpurun_out/r2_search_bert_64.json 2>&1
for f in r2_search_vgg16 r2_search_bert_1 r2_search_bert_16 r2_search_bert_64; do grep "^{" gpurun_out/$f.json | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config'], d['seeds_total'], round(d['wall_s'],3), round(d['rank0_device_ms'],1), round(d['rank0_expand_ms'],1), d['rounds'], d['candidates_evaluated'])"; done
