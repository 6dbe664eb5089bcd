#!/bin/bash
# Dev: build libsig_<tag>.so = the main build's objects with inst_c8.cu recompiled under extra flags.
# usage: scripts/variant_c8.sh <tag> "<nvcc -D flags>"
set -e
cd "$(dirname "$0")/.."
tag=$1; shift
obj=/tmp/inst_c8_$tag.o
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --extended-lambda -Xcompiler -fPIC $@ \
     -c paper_2001_00706_b200/csrc/inst_c8.cu -o $obj
objs=$(ls paper_2001_00706_b200/build_obj/*.o | grep -v inst_c8.cu.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2001_00706_b200/libsig_$tag.so $objs $obj
echo paper_2001_00706_b200/libsig_$tag.so
