mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sketch_fft.py -x -q > gpurun_out/s3t_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3t_tests.log
timeout 600 bash tools/ab_obj.sh sketch tools/_variant_sketch_anchor.cu \
  "python tools/sketch_dmma_probe.py 100000 1000 32; python tools/sketch_dmma_probe.py 100000 1000 64" > gpurun_out/s3t_ab.log 2>&1
