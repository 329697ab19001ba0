mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sketch_fft.py tests/test_gpu_graph.py tests/test_gpu_pipeline.py tests/test_gpu_distributed.py -x -q > gpurun_out/s3n_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3n_tests.log
timeout 900 python bench.py --m 1048576 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s3n_bench.json 2> gpurun_out/s3n_bench.err
