#!/bin/bash
# same-box A/B of library variants: default build vs paper_2209_12769_b200/_build/var/<name>/libdiscob200.so
R=$PWD/paper_2209_12769_b200/_build/var
for r in 1 2 3; do for lib in default "$@"; do
  if [ "$lib" = default ]; then unset FO_LIB_PATH; else export FO_LIB_PATH=$R/$lib/libdiscob200.so; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$lib', 'bench', round(d['value']), 'e2e', round(d['e2e']['value']), {k: round(v, 4) for k, v in d['estimator_roofline']['phase_ms'].items()})"
done; done
for lib in default "$@"; do
  if [ "$lib" = default ]; then unset FO_LIB_PATH; else export FO_LIB_PATH=$R/$lib/libdiscob200.so; fi
  echo "== $lib"; timeout 300 python tools/time_latency.py bert:1 resnet50:1024 gpt2m:1 2>&1 | tail -4
done
