#!/bin/bash
# the other BASELINE.json configs on the current build
timeout 300 python tools/bench_search.py --config vgg16 --seeds 1 > gpurun_out/r2_search_vgg16.json 2>&1
timeout 600 python tools/bench_search.py --config bert --seeds 1 > gpurun_out/r2_search_bert_1.json 2>&1
timeout 600 python tools/bench_search.py --config bert --seeds 64 --oracle-seeds 0 > gpurun_out/r2_search_bert_64.json 2>&1
timeout 900 python tools/bench_configs.py gpt2-sweep > gpurun_out/r2_gpt2m_sweep.json 2>&1
timeout 900 python tools/bench_configs.py synth50k > gpurun_out/r2_synth50k.json 2>&1
for f in r2_search_vgg16 r2_search_bert_1 r2_search_bert_64 r2_gpt2m_sweep r2_synth50k; do echo "== $f"; tail -c 700 gpurun_out/$f.json; echo; done
