#!/bin/bash
# shared-memory ready rings in the warp geometry (FO_RING_SMEM) A/B + parity
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -1
for r in 1 2; do for m in 0 1; do
  FO_RING_SMEM=$m timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('ring_smem=$m', 'bench', round(d['value']), 'e2e', round(d['e2e']['value']), d['estimator_roofline']['phase_ms'])"
done; done
FO_RING_SMEM=1 python tools/time_latency.py fp64 resnet50:1024 resnet50:2048 bert:4096 2>&1 | tail -3
