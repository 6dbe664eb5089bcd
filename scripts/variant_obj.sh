#!/bin/bash
# Dev: build libsig_<tag>.so = the main build's objects with the named sources recompiled under extra
# flags.  usage: scripts/variant_obj.sh <tag> "<src1.cu src2.cu ...>" [nvcc flags...]
set -e
cd "$(dirname "$0")/.."
tag=$1; shift
srcs=$1; shift
objs=""
skip=""
for s in $srcs; do
  o=/tmp/var_${tag}_$s.o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --extended-lambda -Xcompiler -fPIC \
       -Xptxas -warn-spills "$@" -c paper_2001_00706_b200/csrc/$s -o $o &
  objs="$objs $o"
  skip="$skip|/$s.o"
done
wait
base=$(ls paper_2001_00706_b200/build_obj/*.o | grep -vE "(${skip#|})$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2001_00706_b200/libsig_$tag.so $base $objs
echo paper_2001_00706_b200/libsig_$tag.so
