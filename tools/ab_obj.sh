#!/bin/bash
# A/B one translation unit: tools/ab_obj.sh <obj-name> <variant.cu> "<timing command>"
# Relinks the library with the variant object in place of build/<obj-name>.o, runs the
# timing command, then restores the current build and runs it again.
set -e
NVCC="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Ipaper_2603_16644_b200/csrc"
cp paper_2603_16644_b200/libsklsq.so /tmp/libsklsq.base.so
objs=$(ls paper_2603_16644_b200/csrc/*.cu | xargs -n1 basename | sed "s/\.cu$/.o/" | grep -v "^$1.o$" | sed "s|^|build/|" | tr '\n' ' ')
$NVCC -c "$2" -o /tmp/variant.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2603_16644_b200/libsklsq.so $objs /tmp/variant.o -cudart static
echo "== variant $2"; bash -c "$3"
cp /tmp/libsklsq.base.so paper_2603_16644_b200/libsklsq.so
echo "== current"; bash -c "$3"
