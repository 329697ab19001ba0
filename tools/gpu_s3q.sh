mkdir -p gpurun_out
timeout 900 python tools/latency_breakdown.py --m 100000 --n 1000 --kappa 1e10 --method pne --precision single --reps 10 > gpurun_out/s3q_lat_c2_pne.json 2> gpurun_out/s3q_lat_c2_pne.err
timeout 900 python tools/latency_breakdown.py --m 100000 --n 1000 --kappa 1e10 --method hpne --precision single --reps 10 > gpurun_out/s3q_lat_c2_hpne.json 2> gpurun_out/s3q_lat_c2_hpne.err
