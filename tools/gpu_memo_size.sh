#!/bin/bash
# estimator memo size A/B (FO_MEMO_LOG2 = log2 slots per precision; 32 B per slot)
for r in 1 2; do for m in 20 18 17 16; do
  FO_MEMO_LOG2=$m timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('log2=$m', 'bench', round(d['value']), 'e2e', round(d['e2e']['value']), d['estimator_roofline']['phase_ms'])"
done; done
