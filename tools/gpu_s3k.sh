mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_graph.py tests/test_gpu_pipeline.py -x -q > gpurun_out/s3k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3k_tests.log
for m in pne hpne; do timeout 300 python tools/latency_breakdown.py --method $m > gpurun_out/s3k_lat_$m.json 2> gpurun_out/s3k_lat_$m.err; done
