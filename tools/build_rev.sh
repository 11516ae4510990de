#!/bin/bash
# Build libstreamflow.so from the sources of git revision <rev> into build_<name>/ (A/B against an
# earlier kernel on the same box):  tools/build_rev.sh <name> <rev> [patch.py]
# (patch.py, if given, runs with the extracted tree as its working directory before the build)
set -e
name=$1; rev=$2; patch=${3:-}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
src=$(mktemp -d)
git -C $ROOT archive $rev paper_2511_22009_b200/csrc include | tar -x -C $src
if [ -n "$patch" ]; then (cd $src && python $ROOT/$patch); fi
out=$ROOT/build_$name
mkdir -p $out
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O3 -I $src/include"
objs=""
for f in $src/paper_2511_22009_b200/csrc/*.cu; do
  obj=$out/$(basename ${f%.cu}).o
  nvcc $FLAGS -c $f -o $obj &
  objs="$objs $obj"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -o $out/libstreamflow.so $objs -Xlinker -rpath=/usr/local/cuda/lib64
rm -rf $src
echo $out/libstreamflow.so
