#!/bin/bash
# A/B of the extended L2 discards (FO_L2_DISCARD): bench value + DRAM bytes per launch
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -1
for r in 1 2; do for d in 0 1; do
  FO_L2_DISCARD=$d timeout 300 python bench.py --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('discard=$d', 'bench', round(d['value']), 'e2e', round(d['e2e']['value']), d['estimator_roofline']['phase_ms'])"
done; done
for d in 0 1; do
  FO_L2_DISCARD=$d timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:score_kernel -c 2 python tools/prof_score.py resnet50 4096 fp32 2 2>&1 | grep -E "dram__|gpu__time|lts__" | sed "s/^/discard=$d /"
done
