mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_qr_blocked.py tests/test_gpu_graph.py -x -q > gpurun_out/s3d_qr_graph.log 2>&1; echo "rc=$?" >> gpurun_out/s3d_qr_graph.log
for m in hpne pne; do timeout 300 python tools/latency_breakdown.py --method $m > gpurun_out/s3d_lat_$m.json 2> gpurun_out/s3d_lat_$m.err; done
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s3d_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3d_gpu_tests.log
