mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sketch_fft.py -x -q > gpurun_out/s2d_tests.log 2>&1; tail -2 gpurun_out/s2d_tests.log
SK_FFT_PROFILE=1 timeout 300 python tools/bench_sketch.py --levels 16,32,64 --algos fft --reps 2 > gpurun_out/s2d.json 2> gpurun_out/s2d.err
cat gpurun_out/s2d.json; grep 'sketch_fft M=' gpurun_out/s2d.err | tail -6
