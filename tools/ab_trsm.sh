#!/bin/bash
# A/B TRSM kernel variants (K-step depth x ring stages): compile each variant object
# with -DSK_TRSM_BK/-DSK_TRSM_STAGES, relink the library, time the 4M x 2048 TRSM.
# Usage: tools/ab_trsm.sh "8 6" "32 2" ...   (run on the GPU box after `make`)
set -e
NVCC="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
cp paper_2603_16644_b200/libsklsq.so /tmp/libsklsq.base.so
objs=$(ls paper_2603_16644_b200/csrc/*.cu | xargs -n1 basename | sed "s/\.cu$/.o/" | grep -v "^trsm.o$" | sed "s|^|build/|" | tr '\n' ' ')
for v in "$@"; do
  set -- $v
  $NVCC -DSK_TRSM_BK=$1 -DSK_TRSM_STAGES=$2 -c paper_2603_16644_b200/csrc/trsm.cu -o /tmp/trsm_v.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2603_16644_b200/libsklsq.so $objs /tmp/trsm_v.o -cudart static
  echo "== BK=$1 STAGES=$2"; python tools/trsm_split.py 2048
done
cp /tmp/libsklsq.base.so paper_2603_16644_b200/libsklsq.so
echo "== base"; python tools/trsm_split.py 2048
