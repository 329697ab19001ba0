#!/bin/bash
# A/B the TRSM kernel under extra compile flags: tools/ab_trsm_flags.sh "-DSK_TRSM_NOSUB" ...
# (relinks the library per variant, times the 4M x 2048 TRSM, restores the build)
set -e
NVCC="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
cp paper_2603_16644_b200/libsklsq.so /tmp/libsklsq.base.so
objs=$(ls paper_2603_16644_b200/csrc/*.cu | xargs -n1 basename | sed "s/\.cu$/.o/" | grep -v "^trsm.o$" | sed "s|^|build/|" | tr '\n' ' ')
for v in "$@"; do
  $NVCC $v -c paper_2603_16644_b200/csrc/trsm.cu -o /tmp/trsm_v.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2603_16644_b200/libsklsq.so $objs /tmp/trsm_v.o -cudart static
  echo "== $v"; python tools/trsm_split.py 2048
done
cp /tmp/libsklsq.base.so paper_2603_16644_b200/libsklsq.so
echo "== base"; python tools/trsm_split.py 2048
