#!/bin/bash
# Round-2 GPU pass: the -m gpu suite, smoke, the bench (both arms).
# Usage (from the repo root, under gpurun): bash tools/gpu_r2_full.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
tail -3 gpurun_out/${TAG}_pytest_gpu.log
cat gpurun_out/${TAG}_smoke.log | tail -2
head -c 600 gpurun_out/${TAG}_bench.json; echo
head -c 300 gpurun_out/${TAG}_bench_ref.json; echo
