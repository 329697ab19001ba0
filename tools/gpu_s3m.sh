mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sketch_fft.py -x -q > gpurun_out/s3m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3m_tests.log
timeout 900 bash tools/ab_obj.sh sketch_fft tools/_variant_sketch_fft_old.cu \
  "python tools/bench_sketch.py --levels 16,64 --algos fft --reps 5" > gpurun_out/s3m_ab.log 2>&1
