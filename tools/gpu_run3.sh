timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -3
timeout 300 python tools/bench_search.py --config vgg16 --seeds 1 2>&1 | tail -1
timeout 300 python tools/bench_search.py --config bert --seeds 1 --oracle-seeds 1 2>&1 | tail -1
timeout 300 python tools/bench_search.py --config bert --seeds 16 --oracle-seeds 0 2>&1 | tail -1
timeout 600 python tools/bench_search.py --config bert --seeds 256 --oracle-seeds 0 2>&1 | tail -1
timeout 900 python tools/bench_configs.py synth50k --batch 8192 --distinct 8192 2>&1 | tail -1
