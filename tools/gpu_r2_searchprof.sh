#!/bin/bash
# single-seed search latency breakdown (FO_SEARCH_PROFILE), warm handle, VGG-16 and BERT
TAG=${1:-sp}
mkdir -p gpurun_out
export FO_SEARCH_PROFILE=1
for c in vgg16 bert; do
  timeout 300 python tools/bench_search.py --config $c --seeds 1 --oracle-seeds 0 > gpurun_out/${TAG}_$c.json 2> gpurun_out/${TAG}_$c.err
  tail -c 600 gpurun_out/${TAG}_$c.json; echo; grep fo_search_run gpurun_out/${TAG}_$c.err
done
timeout 300 python tools/search_latency.py > gpurun_out/${TAG}_lat.txt 2>&1; cat gpurun_out/${TAG}_lat.txt
