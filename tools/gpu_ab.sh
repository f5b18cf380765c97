# A/B: default lib vs variant libs given as args
for lib in default "$@"; do
  if [ "$lib" = default ]; then unset FO_LIB_PATH; else export FO_LIB_PATH=$PWD/_variants/$lib/libdiscob200.so; fi
  for c in "resnet50 4096" "bert 4096" "vgg16 4096" "resnet50 4096 fp64"; do timeout 120 python tools/time_score.py $c; done
  timeout 300 python tools/time_latency.py bert:1 bert:148 resnet50:1 resnet50:512 resnet50:1024 resnet50:2048 resnet50:4096 gpt2m:1
done
