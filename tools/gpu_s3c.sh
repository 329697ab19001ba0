mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_graph.py -x -q > gpurun_out/s3c_graph_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3c_graph_tests.log
for m in hpne pne; do timeout 300 python tools/latency_breakdown.py --method $m > gpurun_out/s3c_lat_$m.json 2> gpurun_out/s3c_lat_$m.err; done
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_graph.py > gpurun_out/s3c_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3c_gpu_tests.log
