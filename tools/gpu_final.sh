# round-end measurement pass (1 GPU): tests, bench line, reference arm, launch
# list, one ncu --set full capture of the score kernel (bench's sparse config),
# search and config benches
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/final_pytest_gpu.log 2>&1; tail -2 gpurun_out/final_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -c 600 gpurun_out/final_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_bench_ref.json 2>&1; tail -c 300 gpurun_out/final_bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final_ncu_launch.log 2>&1; echo launches rc=$?
FO_PROF_ENCODING=delta timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_kernel -c 1 -o gpurun_out/final_score -f python tools/prof_score.py resnet50 4096 fp32 1 > gpurun_out/final_ncu_full.log 2>&1; echo full rc=$?
timeout 300 python tools/bench_search.py --config vgg16 --seeds 1 > gpurun_out/final_search.jsonl 2>&1
timeout 300 python tools/bench_search.py --config bert --seeds 1 >> gpurun_out/final_search.jsonl 2>&1
timeout 300 python tools/bench_search.py --config bert --seeds 16 --oracle-seeds 2 >> gpurun_out/final_search.jsonl 2>&1
timeout 600 python tools/bench_search.py --config bert --seeds 64 --oracle-seeds 0 >> gpurun_out/final_search.jsonl 2>&1
timeout 900 python tools/bench_search.py --config bert --seeds 256 --oracle-seeds 0 >> gpurun_out/final_search.jsonl 2>&1
timeout 900 python tools/bench_configs.py gpt2-sweep --batch 512 > gpurun_out/final_gpt2m.json 2>&1
timeout 900 python tools/bench_configs.py synth50k --batch 8192 > gpurun_out/final_synth50k.json 2>&1
timeout 300 python tools/time_latency.py bert:1 vgg16:1 resnet50:1 gpt2m:1 resnet50:512 > gpurun_out/final_latency.jsonl 2>&1
grep -h "{" gpurun_out/final_search.jsonl | cut -c1-200
