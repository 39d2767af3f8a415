#!/bin/bash
# Build an alternative libpcirc_b200.so with extra -D flags for one source
# (kernel A/B experiments, loaded with PCB_LIB=...):
#   tools/build_variant.sh <out.so> <source.cu> -DNAME=VALUE ...
set -eu
out=$1; src=$2; shift 2
L=paper_2406_00766_b200/_lib
objs=()
for o in $L/*.o; do
  [ "$(basename $o .o)" = "$(basename $src .cu)" ] || objs+=("$o")
done
tmpo=$(mktemp --suffix=.o)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC "$@" \
  -c paper_2406_00766_b200/csrc/$src -o $tmpo
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out "${objs[@]}" $tmpo -lcudart
rm -f $tmpo
