# FFT: parity, then pass split per level with prefetch on/off, with and without expandable segments.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sketch_fft.py -x -q > gpurun_out/s2c_tests.log 2>&1; tail -2 gpurun_out/s2c_tests.log
for pf in 0 1; do
  SK_FFT_PF=$pf SK_FFT_PROFILE=1 timeout 300 python tools/bench_sketch.py --levels 16,32 --algos fft --reps 2 > gpurun_out/s2c_pf$pf.json 2> gpurun_out/s2c_pf$pf.err
  echo "PF=$pf"; cat gpurun_out/s2c_pf$pf.json; grep 'sketch_fft M=' gpurun_out/s2c_pf$pf.err | tail -2
done
PYTORCH_CUDA_ALLOC_CONF= SK_FFT_PROFILE=1 timeout 300 python tools/bench_sketch.py --levels 32,64 --algos fft --reps 2 > gpurun_out/s2c_noexp.json 2> gpurun_out/s2c_noexp.err
echo "no expandable"; cat gpurun_out/s2c_noexp.json; grep 'sketch_fft M=' gpurun_out/s2c_noexp.err | tail -4
