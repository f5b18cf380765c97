for lib in unroll stop1 stop2 stop3; do
  export FO_LIB_PATH=$PWD/_variants/$lib/libdiscob200.so
  echo "== $lib"
  timeout 300 python tools/time_latency.py bert:1 resnet50:1 vgg16:1 gpt2m:1 resnet50:4096
done
python - <<'PY'
import paper_2209_12769_b200 as P
for c in ["bert","resnet50","vgg16","gpt2m"]:
    g=P.load_workload(c)[0]
    print(c, len(g.ops), sum(len(o.inputs) if hasattr(o,'inputs') else 0 for o in g.ops), len(g.allreduces))
PY
