#!/bin/bash
# Build an experimental libtofu variant with extra nvcc defines: tools/build_variant.sh OUT.so -DNAME=VAL ...
set -e
OUT=$1; shift
cd "$(dirname "$0")/.."
P=paper_1807_08887_b200
mkdir -p /tmp/tofu_variant
objs=()
for f in $P/csrc/cuda/*.cu; do
  o=/tmp/tofu_variant/$(basename $f).o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I include -I $P/csrc "$@" -c $f -o $o &
  objs+=($o)
done
for f in $P/csrc/host/*.cpp; do
  o=/tmp/tofu_variant/$(basename $f).o
  nvcc -O3 -std=c++17 -Xcompiler -fPIC -I include -I $P/csrc -x c++ -c $f -o $o &
  objs+=($o)
done
for p in $(jobs -p); do wait $p || { echo "compile failed"; exit 1; }; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $OUT "${objs[@]}" -ldl -lpthread -lrt
echo built $OUT
