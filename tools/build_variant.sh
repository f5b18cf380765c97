# build a variant library from _variants/<name>/ (files there override csrc/)
set -e
d=_variants/$1
for f in paper_2209_12769_b200/csrc/*; do b=$(basename $f); [ -f $d/$b ] || cp $f $d/$b; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-fopenmp,-O3 -shared \
  -I include $d/score.cu $d/capi.cu $d/engine.cpp -o $d/libdiscob200.so -lgomp ${@:2}
