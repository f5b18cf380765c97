# multi-GPU scaling on one box: bench.py (batch sharding) and the sharded search
for n in 1 2 4; do
  if [ $n = 1 ]; then timeout 600 python bench.py --no-cpu-baseline > gpurun_out/scale_$n.json 2>gpurun_out/scale_$n.err;
  else timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --no-cpu-baseline > gpurun_out/scale_$n.json 2>gpurun_out/scale_$n.err; fi
  tail -1 gpurun_out/scale_$n.json | cut -c1-300
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 tools/bench_search.py --config bert --seeds 64 --oracle-seeds 0 > gpurun_out/scale_search4.json 2>gpurun_out/scale_search4.err; tail -1 gpurun_out/scale_search4.json | cut -c1-400
