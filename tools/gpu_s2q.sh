timeout 900 python -m pytest tests/test_gpu_sketch_fft.py -x -q > gpurun_out/s2q_tests.log 2>&1; tail -2 gpurun_out/s2q_tests.log
for cb in 1 0; do
SK_FFT_CB32=$cb SK_FFT_PROFILE=1 timeout 300 python tools/bench_sketch.py --levels 16 --algos fft --reps 3 > gpurun_out/s2q_$cb.json 2> gpurun_out/s2q_$cb.err
echo cb32=$cb; cat gpurun_out/s2q_$cb.json; grep 'sketch_fft M=' gpurun_out/s2q_$cb.err | tail -2
done
