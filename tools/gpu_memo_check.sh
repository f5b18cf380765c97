#!/bin/bash
# epoch memo: full GPU tests, bench x2, e2e parts
timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -1
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('bench', round(d['value']), 'e2e', round(d['e2e']['value']), d['ms_per_step'])"; done
python tools/time_e2e_parts.py 2>&1 | tail -6
