# CUDA-graph plan (deferred verdicts) + latency; QR per-call env paths; sketch pass-A 32-bit item decode A/B
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_graph.py -x -q > gpurun_out/s3a_graph_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3a_graph_tests.log
for m in hpne pne; do timeout 300 python tools/latency_breakdown.py --method $m > gpurun_out/s3a_lat_$m.json 2> gpurun_out/s3a_lat_$m.err; done
timeout 900 python -m pytest tests/test_gpu_qr_blocked.py tests/test_gpu_qr_smem.py tests/test_gpu_sketch_fft.py -x -q > gpurun_out/s3a_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s3a_tests.log
timeout 600 bash tools/ab_obj.sh sketch_fft tools/_variant_sketch_fft_old.cu \
  "python tools/bench_sketch.py --levels 16,32,64 --algos fft --reps 5" > gpurun_out/s3a_ab.log 2>&1
for b in 32 64; do timeout 300 python tools/qr_probe.py 6144 2048 $b >> gpurun_out/s3a_qr.jsonl 2>>gpurun_out/s3a_qr.err; done
