#!/bin/bash
for b in 100 130; do FO_WS_BUDGET_GB=$b timeout 300 python tools/bench_configs.py synth50k 2>&1 | grep "^{" | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('budget', $b, 'GB', round(d['value']), 'cand/s', round(d['ms_per_round'],1), 'ms/round', d['oracle_check'])"; done
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
