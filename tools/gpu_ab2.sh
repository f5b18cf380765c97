# A/B of event-loop variants: latency (both geometries) and throughput
for lib in default "$@"; do
  if [ "$lib" = default ]; then unset FO_LIB_PATH; else export FO_LIB_PATH=$PWD/_variants/$lib/libdiscob200.so; fi
  echo "== $lib"
  for c in "resnet50 4096" "bert 4096" "resnet50 4096 fp64"; do timeout 120 python tools/time_score.py $c | cut -c1-200; done
  timeout 300 python tools/time_latency.py bert:1 resnet50:1 vgg16:1 gpt2m:1 resnet50:512
done
