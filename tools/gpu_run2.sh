timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -3
timeout 900 python tools/bench_configs.py gpt2-sweep --batch 512 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); d.pop('rows'); print(json.dumps(d))"
