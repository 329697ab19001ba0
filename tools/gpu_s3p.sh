mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_graph.py tests/test_gpu_ozaki.py tests/test_gpu_trsm_ozaki.py tests/test_gpu_pipeline.py tests/test_gpu_kernels.py -x -q > gpurun_out/s3p_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3p_tests.log
timeout 900 python bench.py --m 1048576 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s3p_bench.json 2> gpurun_out/s3p_bench.err
