#!/bin/bash
# A/B the TRSM leaf's rows per CTA (SK_TRSM_BMR 128 default vs 64: 3 CTAs/SM), leaf width 1024 and 512.
NVCC="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
cp paper_2603_16644_b200/libsklsq.so /tmp/libsklsq.base.so
objs=$(ls paper_2603_16644_b200/csrc/*.cu | xargs -n1 basename | sed "s/\.cu$/.o/" | grep -v "^trsm.o$" | sed "s|^|build/|" | tr '\n' ' ')
run() { for b in 1024 512; do SK_TRSM_OZ_BASE=$b SK_TRSM_OZ_PROFILE=1 python tools/trsm_oz_probe.py 4194304 2048 2 2>&1 | grep -E '"ozaki"|trsm_ozaki' | tail -2 | sed "s/^/base=$b /"; done; }
echo "== BMR=128"; run
$NVCC -DSK_TRSM_BMR=64 -c paper_2603_16644_b200/csrc/trsm.cu -o /tmp/trsm_v.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2603_16644_b200/libsklsq.so $objs /tmp/trsm_v.o -cudart static
echo "== BMR=64"; run
timeout 600 python -m pytest tests/test_gpu_trsm_ozaki.py tests/test_gpu_kernels.py -x -q -k "trsm" 2>&1 | tail -2
cp /tmp/libsklsq.base.so paper_2603_16644_b200/libsklsq.so
