mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_pass_b_tf32 -c 1 -o gpurun_out/s2h_ncu -f \
  python tools/bench_sketch.py --m 4194304 --n 256 --levels 16 --algos fft --reps 1 > gpurun_out/s2h_ncu.log 2>&1
ncu -i gpurun_out/s2h_ncu.ncu-rep --page details --csv > gpurun_out/s2h_details.csv 2>/dev/null
ncu -i gpurun_out/s2h_ncu.ncu-rep --page source --csv --print-source sass > gpurun_out/s2h_src.csv 2>/dev/null
rm -f gpurun_out/s2h_ncu.ncu-rep
