#!/bin/bash
# Dev: build libsig_<tag>.so = the main build's objects with api.cu recompiled under extra flags.
set -e
cd "$(dirname "$0")/.."
tag=$1; shift
obj=/tmp/api_$tag.o
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --extended-lambda -Xcompiler -fPIC $@ \
     -c paper_2001_00706_b200/csrc/api.cu -o $obj
objs=$(ls paper_2001_00706_b200/build_obj/*.o | grep -v "/api.cu.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2001_00706_b200/libsig_$tag.so $objs $obj
echo paper_2001_00706_b200/libsig_$tag.so
