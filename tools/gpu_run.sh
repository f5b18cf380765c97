#!/bin/bash
# GPU measurement suites (run from the repo root on a B200 box, e.g. under
# gpurun).  Outputs go to gpurun_out/<TAG>_*; the summaries worth keeping are
# copied to profiles/ by hand.
#
#   bash tools/gpu_run.sh tests    [TAG]   # -m gpu suite + smoke
#   bash tools/gpu_run.sh bench    [TAG]   # bench.py, both arms, clocks
#   bash tools/gpu_run.sh launches [TAG]   # bench.py's launch list under ncu (per-launch times)
#   bash tools/gpu_run.sh profile  [TAG]   # phase timings + ncu --set full of the three incremental kernels
#   bash tools/gpu_run.sh configs  [TAG]   # BASELINE configs[0], [2] searches, [3] sweep, [4] synth50k
#   bash tools/gpu_run.sh scale    [TAG]   # 2 / 4 GPUs: bench, synth50k, BERT 256-seed search (gpurun --gpus 4)
#   bash tools/gpu_run.sh multirank [TAG]  # two-rank exchange tests (the NCCL ones need gpurun --gpus 2)
#   bash tools/gpu_run.sh ab-snap  [TAG]   # K3 fast-forward on / off, bit-exactness
#   bash tools/gpu_run.sh ab-submit [TAG]  # pipelined submissions on 3 / 2 / 1 compute streams (e2e)
#   bash tools/gpu_run.sh ab-snap-bench [TAG]  # bench figures (pipelined, e2e, serial) with / without the K3 fast-forward
#   bash tools/gpu_run.sh ab-tc    [TAG]   # tensor-core MP transforms: error and K2 time
#   bash tools/gpu_run.sh ab-exchange [TAG]  # 4 GPUs: per-round exchange (native / torch thread) vs once
#   bash tools/gpu_run.sh search-latency [TAG]  # single-seed search breakdown (FO_SEARCH_PROFILE)
SUITE=${1:?suite}
TAG=${2:-$SUITE}
O=gpurun_out/${TAG}
mkdir -p gpurun_out
case $SUITE in
tests)
  timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -x > ${O}_pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> ${O}_pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > ${O}_smoke.log 2>&1
  echo "smoke rc=$?" >> ${O}_smoke.log
  tail -3 ${O}_pytest_gpu.log; tail -2 ${O}_smoke.log
  ;;
bench)
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > ${O}_smi.txt 2>&1
  timeout 900 python bench.py > ${O}_bench.json 2> ${O}_bench.err
  timeout 600 python bench.py --impl reference > ${O}_bench_ref.json 2> ${O}_bench_ref.err
  head -c 600 ${O}_bench.json; echo; head -c 300 ${O}_bench_ref.json; echo
  ;;
launches)
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file ${O}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-search > ${O}_under_ncu.log 2>&1
  grep -E "score_kernel|fo::" ${O}_launches.csv | cut -c1-160 | head -12
  ;;
profile)
  for c in "resnet50 4096" "bert 4096" "vgg16 4096"; do timeout 90 python tools/time_inc.py $c; done > ${O}_time.jsonl 2> ${O}_time.err
  cat ${O}_time.jsonl
  for k in "score_kernel_inc_k3:k3" "score_kernel_inc_mp:mp" "score_kernel_inc:setup"; do
    rx=${k%%:*}; nm=${k##*:}
    if [ $nm = setup ]; then f="-k $rx"; else f="-k regex:$rx"; fi
    timeout 300 ncu --set full --import-source on --clock-control none $f -s 2 -c 1 -o ${O}_$nm \
      python tools/prof_score.py resnet50 4096 fp32 3 > ${O}_ncu_$nm.log 2>&1
    tail -1 ${O}_ncu_$nm.log
  done
  ;;
configs)
  timeout 300 python tools/bench_search.py --config vgg16 --seeds 1 > ${O}_search_vgg16.json 2>&1
  timeout 600 python tools/bench_search.py --config bert --seeds 1 > ${O}_search_bert_1.json 2>&1
  timeout 600 python tools/bench_search.py --config bert --seeds 16 --oracle-seeds 0 > ${O}_search_bert_16.json 2>&1
  timeout 600 python tools/bench_search.py --config bert --seeds 64 --oracle-seeds 0 > ${O}_search_bert_64.json 2>&1
  timeout 900 python tools/bench_configs.py gpt2-sweep --batch 512 > ${O}_gpt2m_sweep.json 2>&1
  timeout 900 python tools/bench_configs.py synth50k > ${O}_synth50k.json 2>&1
  for f in search_vgg16 search_bert_1 search_bert_16 search_bert_64 gpt2m_sweep synth50k; do
    echo "== $f"; grep "^{" ${O}_$f.json | tail -1 | head -c 500; echo
  done
  ;;
scale)
  for n in 2 4; do
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n \
      bench.py --gpus $n --steps 20 --warmup 5 2>/dev/null | grep "^{" > ${O}_bench_${n}gpu.json
    head -c 400 ${O}_bench_${n}gpu.json; echo
  done
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29520 \
    tools/bench_configs.py synth50k 2>/dev/null | grep "^{" > ${O}_synth50k_4gpu.json
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 \
    tools/bench_search.py --config bert --seeds 64 --oracle-seeds 0 2>/dev/null | grep "^{" > ${O}_search_bert256_4gpu.json
  tail -c 300 ${O}_synth50k_4gpu.json; echo; tail -c 400 ${O}_search_bert256_4gpu.json; echo
  ;;
multirank)
  nvidia-smi -L
  timeout 800 python -m pytest tests/test_gpu_multirank.py -q -x --timeout 300 > ${O}_multirank.log 2>&1
  echo "rc=$?" >> ${O}_multirank.log; tail -3 ${O}_multirank.log
  ;;
ab-snap)
  timeout 400 python tools/time_snap.py resnet50,bert,vgg16 4096 > ${O}_ab.jsonl 2> ${O}_ab.err
  timeout 200 python tools/time_snap.py resnet50 4096 fp64 >> ${O}_ab.jsonl 2>> ${O}_ab.err
  cat ${O}_ab.jsonl
  ;;
ab-submit)
  for rep in 1 2; do for v in 3 2 1; do
    export FO_SUBMIT_STREAMS=$v
    echo "streams=$v $(timeout 300 python bench.py --no-cpu-baseline --no-search --steps 20 --warmup 5 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["e2e"]["synchronous_value"])')"
  done; done | tee ${O}_ab.txt
  unset FO_SUBMIT_STREAMS
  ;;
ab-snap-bench)
  for rep in 1 2; do for v in 0 1; do
    if [ $v = 1 ]; then export FO_INC_NO_SNAP=1; else unset FO_INC_NO_SNAP; fi
    echo "no_snap=$v $(timeout 300 python bench.py --no-cpu-baseline --no-search --steps 40 --warmup 5 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["serial"]["value"])')"
  done; done | tee ${O}_ab.txt
  unset FO_INC_NO_SNAP
  ;;
ab-tc)
  timeout 300 python -m pytest tests/test_gpu_tensorcore.py -q -x --timeout 250 > ${O}_tc_test.log 2>&1; tail -3 ${O}_tc_test.log
  for c in resnet50 bert; do timeout 200 python tools/time_mp_arith.py $c 4096; done > ${O}_tc_time.jsonl 2>&1
  cat gpurun_out/tensorcore_error.json ${O}_tc_time.jsonl
  ;;
ab-exchange)
  : > ${O}_variants.jsonl
  for rep in 1 2; do
    for v in "end 0 0" "round 8 0" "round 8 1"; do
      set -- $v
      if [ $3 = 1 ]; then export FO_XCHG_PY=1; else unset FO_XCHG_PY; fi
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 \
        tools/bench_search.py --config bert --seeds 64 --oracle-seeds 0 --exchange $1 --lag $2 2>/dev/null \
        | grep '"metric"' | sed "s/}\$/, \"py\": $3}/" >> ${O}_variants.jsonl
    done
  done
  unset FO_XCHG_PY
  cat ${O}_variants.jsonl | cut -c1-300
  ;;
search-latency)
  FO_SEARCH_PROFILE=1 timeout 300 python tools/search_latency.py vgg16,bert > ${O}_lat.txt 2>&1
  cat ${O}_lat.txt
  ;;
*)
  echo "unknown suite $SUITE"; exit 2
  ;;
esac
