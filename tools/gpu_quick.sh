# parity suite + latency/throughput snapshot of the current build
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 2>&1 | tail -2
timeout 300 python tools/time_latency.py bert:1 bert:148 vgg16:1 resnet50:1 resnet50:512 resnet50:640 gpt2m:1
for c in "resnet50 4096" "bert 4096" "vgg16 4096" "resnet50 4096 fp64"; do timeout 120 python tools/time_score.py $c; done
