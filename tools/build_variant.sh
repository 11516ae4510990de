#!/bin/bash
# Build libstreamflow.so with extra nvcc defines into build_<name>/ for same-box A/B runs:
#   tools/build_variant.sh <name> -DFOO=1 ...   ->  SF_LIB_PATH=build_<name>/libstreamflow.so python ...
set -e
name=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
out=$ROOT/build_$name
mkdir -p $out
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O3 -I $ROOT/include"
objs=""
for src in $ROOT/paper_2511_22009_b200/csrc/*.cu; do
  obj=$out/$(basename ${src%.cu}).o
  nvcc $FLAGS "$@" -c $src -o $obj &
  objs="$objs $obj"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -o $out/libstreamflow.so $objs -Xlinker -rpath=/usr/local/cuda/lib64
echo $out/libstreamflow.so
