#!/bin/bash
# Build libsf_<name>.so with extra nvcc flags for one source (diagnostic variants):
#   tools/build_variant.sh <name> <source.cu> [nvcc flags...]
set -e
NAME=$1; SRC=$2; shift 2
ROOT=$(cd $(dirname $0)/.. && pwd)
B=$ROOT/build/var_$NAME; mkdir -p $B
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O3 -I $ROOT/include"
objs=""
for f in $ROOT/paper_2511_22009_b200/csrc/*.cu; do
  bn=$(basename $f .cu)
  if [ "$bn" == "$(basename $SRC .cu)" ]; then
    nvcc $FLAGS "$@" -c $f -o $B/$bn.o
  else
    cp $ROOT/build/$bn.o $B/$bn.o
  fi
  objs="$objs $B/$bn.o"
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -o $ROOT/paper_2511_22009_b200/libsf_$NAME.so $objs -Xlinker -rpath=/usr/local/cuda/lib64
echo built libsf_$NAME.so
