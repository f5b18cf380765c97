#!/bin/bash
# K3 A/B: parity tests, headline bench, per-phase latency
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_features.py -q -x -m gpu 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('bench', round(d['value']), 'e2e', round(d['e2e']['value']), d['estimator_roofline']['phase_ms'])"; done
python tools/time_latency_phases.py fp64 bert:1 bert:16 resnet50:1 vgg16:1 gpt2m:1 2>&1 | tail -5
