#!/bin/bash
# A/B of two builds of the library on the bench (pipelined, e2e, serial):
#   bash tools/ab_lib.sh OLD.so NEW.so [reps]
A=${1:?old lib}; B=${2:?new lib}; R=${3:-3}
for r in $(seq $R); do for v in A B; do
  if [ $v = A ]; then L=$A; else L=$B; fi
  echo "$v $(FO_LIB_PATH=$L timeout 300 python bench.py --no-cpu-baseline --no-search --steps 40 --warmup 5 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["serial"]["value"])')"
done; done
