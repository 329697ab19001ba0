mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sketch_fft.py -x -q > gpurun_out/s2g_tests.log 2>&1; tail -15 gpurun_out/s2g_tests.log
SK_FFT_PROFILE=1 timeout 300 python tools/bench_sketch.py --levels 16,64 --algos fft --reps 2 > gpurun_out/s2g.json 2> gpurun_out/s2g.err
cat gpurun_out/s2g.json; grep 'sketch_fft M=' gpurun_out/s2g.err | tail -4
SK_FFT_PROFILE=1 timeout 300 python tools/bench_sketch.py --m 1048576 --n 1024 --levels 16,64 --algos fft --reps 2 > gpurun_out/s2g_1m.json 2> gpurun_out/s2g_1m.err
cat gpurun_out/s2g_1m.json; grep 'sketch_fft M=' gpurun_out/s2g_1m.err | tail -2
