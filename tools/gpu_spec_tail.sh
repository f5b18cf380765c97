#!/bin/bash
# tail speculation (FO_SEARCH_SPEC_AT) on the BERT lock-stepped search, plus 1 seed
mkdir -p gpurun_out
for s in 1 16 64 256; do
  for at in 32; do
    FO_SEARCH_SPEC_AT=$at FO_SEARCH_PROFILE=1 timeout 300 python tools/bench_search.py --config bert --seeds $s --oracle-seeds 0 2>gpurun_out/spec_${s}_${at}.err | sed "s/^/at=$at /"
    tail -1 gpurun_out/spec_${s}_${at}.err
  done
done
