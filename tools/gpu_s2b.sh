# FFT pass-A A/B (prefetch on/off) at 4M x 2048 and ncu of both pass-A precisions at 1M x 256.
mkdir -p gpurun_out
for pf in 1 0; do
  SK_FFT_PF=$pf SK_FFT_PROFILE=1 timeout 300 python tools/bench_sketch.py --levels 32 --algos fft --reps 2 > gpurun_out/s2b_pf$pf.json 2> gpurun_out/s2b_pf$pf.err
  echo "PF=$pf"; grep 'sketch_fft M=' gpurun_out/s2b_pf$pf.err | tail -2
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_pass_a -c 2 -o gpurun_out/s2b_ncu_passa -f \
  python tools/bench_sketch.py --m 1048576 --n 256 --levels 32,64 --algos fft --reps 1 > gpurun_out/s2b_ncu.log 2>&1
tail -3 gpurun_out/s2b_ncu.log
ncu -i gpurun_out/s2b_ncu_passa.ncu-rep --page details --csv > gpurun_out/s2b_ncu_details.csv 2>/dev/null
ncu -i gpurun_out/s2b_ncu_passa.ncu-rep --page source --csv --print-source sass > gpurun_out/s2b_ncu_src.csv 2>/dev/null
ls -la gpurun_out/s2b*
