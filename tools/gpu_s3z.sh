mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sketch_fft.py tests/test_gpu_kernels.py -x -q > gpurun_out/s3z_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3z_tests.log
timeout 600 bash tools/ab_obj.sh sketch tools/_variant_sketch_256.cu \
  "python tools/sketch_dmma_probe.py 100000 1000 32; python tools/sketch_dmma_probe.py 100000 1000 64; python tools/sketch_dmma_probe.py 1000 100 32; python tools/sketch_dmma_probe.py 300000 256 64" > gpurun_out/s3z_ab.log 2>&1
