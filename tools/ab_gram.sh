#!/bin/bash
# A/B Gram kernel variants: relink the library with each variant object and time
# SYRK/GEMM at 1M x 2048 (variants: build/gram_<name>.o, compiled with -DSK_GRAM_* flags).
set -e
cp paper_2603_16644_b200/libsklsq.so /tmp/libsklsq.base.so
for v in "$@"; do
  objs=$(ls build/*.o | grep -v "gram" | tr '\n' ' ')
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2603_16644_b200/libsklsq.so $objs build/gram_$v.o -cudart static
  echo "== $v"; python tools/bench_kernels.py --m 1048576 --only syrk,gemm --reps 3
done
cp /tmp/libsklsq.base.so paper_2603_16644_b200/libsklsq.so
echo "== base"; python tools/bench_kernels.py --m 1048576 --only syrk,gemm --reps 3
