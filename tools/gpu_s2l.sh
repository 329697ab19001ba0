mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jacobi.py tests/test_gpu_sketch_fft.py tests/test_gpu_kernels.py -x -q > gpurun_out/s2l_tests.log 2>&1; tail -3 gpurun_out/s2l_tests.log
SK_FFT_PROFILE=1 timeout 300 python tools/bench_sketch.py --levels 16,64 --algos fft --reps 2 > gpurun_out/s2l_sk.json 2> gpurun_out/s2l_sk.err
cat gpurun_out/s2l_sk.json; grep 'sketch_fft M=' gpurun_out/s2l_sk.err | tail -3
timeout 900 python tools/diag_cost.py > gpurun_out/s2l_diag.json 2> gpurun_out/s2l_diag.err; cat gpurun_out/s2l_diag.json
