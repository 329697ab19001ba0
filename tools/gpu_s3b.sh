mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_graph.py -x -q > gpurun_out/s3b_graph_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3b_graph_tests.log
for m in hpne pne; do timeout 300 python tools/latency_breakdown.py --method $m > gpurun_out/s3b_lat_$m.json 2> gpurun_out/s3b_lat_$m.err; done
SK_QR_BLOCKED=0 timeout 300 python tools/latency_breakdown.py --method hpne > gpurun_out/s3b_lat_hpne_flowqr.json 2>/dev/null
