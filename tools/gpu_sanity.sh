# post-rebuild sanity on a fresh box: GPU parity suite, smoke, one bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/sanity_pytest_gpu.log 2>&1; tail -2 gpurun_out/sanity_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/sanity_bench.json 2> gpurun_out/sanity_bench.err; tail -c 400 gpurun_out/sanity_bench.json
