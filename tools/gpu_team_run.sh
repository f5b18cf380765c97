set -x
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 2>&1 | tail -5
FO_TEAM=1 timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 2>&1 | tail -5
timeout 300 python tools/time_latency.py bert:1 bert:16 bert:48 bert:148 bert:296 vgg16:1 vgg16:48 resnet50:1 resnet50:64 resnet50:296 gpt2m:1 gpt2m:64
timeout 300 python tools/time_score.py resnet50 4096 2>&1 | tail -2
