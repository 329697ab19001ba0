mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sketch_fft.py -x -q > gpurun_out/s2f_tests.log 2>&1; tail -2 gpurun_out/s2f_tests.log
SK_FFT_PROFILE=1 timeout 300 python tools/bench_sketch.py --levels 16,64 --algos fft --reps 2 > gpurun_out/s2f.json 2> gpurun_out/s2f.err
cat gpurun_out/s2f.json; grep 'sketch_fft M=' gpurun_out/s2f.err | tail -4
SK_FFT_PF=1 SK_FFT_PROFILE=1 timeout 300 python tools/bench_sketch.py --levels 32 --algos fft --reps 2 > gpurun_out/s2f_pf.json 2> gpurun_out/s2f_pf.err
echo PF1; grep 'sketch_fft M=' gpurun_out/s2f_pf.err | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_pass -c 2 -o gpurun_out/s2f_ncu32 -f \
  python tools/bench_sketch.py --m 1048576 --n 256 --levels 32 --algos fft --reps 1 > gpurun_out/s2f_ncu.log 2>&1
ncu -i gpurun_out/s2f_ncu32.ncu-rep --page details --csv > gpurun_out/s2f_ncu32_details.csv 2>/dev/null
ncu -i gpurun_out/s2f_ncu32.ncu-rep --page source --csv --print-source sass > gpurun_out/s2f_ncu32_src.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:fft_pass -c 2 -o gpurun_out/s2f_ncu64 -f \
  python tools/bench_sketch.py --m 1048576 --n 256 --levels 64 --algos fft --reps 1 > gpurun_out/s2f_ncu64.log 2>&1
ncu -i gpurun_out/s2f_ncu64.ncu-rep --page details --csv > gpurun_out/s2f_ncu64_details.csv 2>/dev/null
ls -la gpurun_out/s2f*
SK_FFT_PROFILE=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s2f_bench_fft.json 2> gpurun_out/s2f_bench_fft.err
SK_SKETCH16=tc timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s2f_bench_tc.json 2> gpurun_out/s2f_bench_tc.err
for f in fft tc; do python -c "
import json; d=json.loads(open('gpurun_out/s2f_bench_$f.json').read().strip().splitlines()[-1])
print('$f', d['value'], {k:round(v['ms'],1) for k,v in d['stages_ms'].items()}, d.get('clocks'))"; done
grep 'sketch_fft M=' gpurun_out/s2f_bench_fft.err | tail -3
