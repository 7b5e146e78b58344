#!/bin/bash
# usage: tools/build_variant.sh NAME "-DFLAG=1 ..."  -> paper_2503_13086_b200/libssr_NAME.so
# (an experiment build of the whole library with extra nvcc defines; objects in /tmp)
set -e
NAME=$1; DEFS=$2
C=paper_2503_13086_b200/csrc; O=/tmp/ssr_variant_$NAME; mkdir -p $O
F="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $DEFS"
pids=()
for f in $C/*.cu; do
  b=$(basename $f .cu); x=""; [ $b = ssr_project ] && x="-fmad=false"
  /usr/local/cuda/bin/nvcc $F $x -c $f -o $O/$b.o & pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2503_13086_b200/libssr_$NAME.so $O/*.o
