#!/bin/bash
# Build libpct variant: scripts/build_variant.sh <name> <file.cu> [-DFOO=1 ...]
# recompiles one translation unit with extra flags, links it with the other
# objects of lib/ into variants/<name>.so (select with PCT_LIB=variants/<name>.so)
set -e
name=$1; tu=$2; shift 2
L=paper_2403_07631_b200/lib; C=paper_2403_07631_b200/csrc
mkdir -p variants/obj_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --fmad=false \
  -Xcompiler -fPIC,-ffp-contract=off,-O2 -I include "$@" -c $C/$tu -o variants/obj_$name/${tu%.cu}.o
objs=""
for o in $L/*.o; do b=$(basename $o); if [ "$b" = "${tu%.cu}.o" ]; then objs="$objs variants/obj_$name/$b"; else objs="$objs $o"; fi; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$name.so $objs -lcudart -Xcompiler -pthread
echo built variants/$name.so
