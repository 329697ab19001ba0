mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_qr_blocked.py tests/test_gpu_graph.py tests/test_gpu_lu_smem.py tests/test_gpu_kernels.py tests/test_gpu_pipeline.py -x -q > gpurun_out/s3j_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3j_tests.log
for m in hpne pne; do timeout 300 python tools/latency_breakdown.py --method $m > gpurun_out/s3j_lat_$m.json 2> gpurun_out/s3j_lat_$m.err; done
timeout 300 python tools/latency_breakdown.py --method hpne --precision double > gpurun_out/s3j_lat_hpne_double.json 2>/dev/null
