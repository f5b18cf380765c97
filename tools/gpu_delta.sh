timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -3
for e in delta int16; do timeout 600 python bench.py --encoding $e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['value']), d['ms_per_step'], 'e2e', round(d['e2e']['value']), d['e2e']['h2d_bytes_per_step'], d['config']['encoding'])"; done
