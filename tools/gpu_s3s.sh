mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sketch_fft.py tests/test_gpu_kernels.py tests/test_gpu_graph.py -x -q > gpurun_out/s3s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3s_tests.log
timeout 600 bash tools/ab_obj.sh sketch tools/_variant_sketch_old.cu \
  "python tools/sketch_dmma_probe.py 100000 1000 32; python tools/sketch_dmma_probe.py 100000 1000 64; python tools/sketch_dmma_probe.py 1000 100 32" > gpurun_out/s3s_ab.log 2>&1
timeout 600 python tools/latency_breakdown.py --m 100000 --n 1000 --kappa 1e10 --method hpne --precision single --reps 10 > gpurun_out/s3s_lat_c2.json 2>/dev/null
