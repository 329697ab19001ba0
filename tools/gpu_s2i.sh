mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sketch_fft.py -x -q > gpurun_out/s2i_tests.log 2>&1; tail -2 gpurun_out/s2i_tests.log
for n in 256 2048; do
SK_FFT_PROFILE=1 timeout 300 python tools/bench_sketch.py --n $n --levels 16,64 --algos fft --reps 2 > gpurun_out/s2i_$n.json 2> gpurun_out/s2i_$n.err
echo "n=$n"; cat gpurun_out/s2i_$n.json; grep 'sketch_fft M=' gpurun_out/s2i_$n.err | tail -3
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
