timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -2
for c in "resnet50 4096" "bert 4096" "vgg16 4096"; do timeout 120 python tools/time_score.py $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], d['K'], round(d['ms_median'],4), d['max_status'], d['cost_sum'])"; done
timeout 300 python tools/time_latency.py bert:1 resnet50:1 gpt2m:1
timeout 300 python tools/ab_retry.py
