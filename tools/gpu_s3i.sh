mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_qr_blocked.py tests/test_gpu_graph.py -x -q > gpurun_out/s3i_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3i_tests.log
timeout 300 python tools/latency_breakdown.py --method hpne > gpurun_out/s3i_lat_hpne.json 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qrb_panel_small -c 1 -o gpurun_out/s3i_ps -f python tools/qr_probe.py 300 100 32 > gpurun_out/s3i_ncu1.log 2>&1
ncu -i gpurun_out/s3i_ps.ncu-rep --page details --csv > gpurun_out/s3i_ps_details.csv 2>/dev/null
ncu -i gpurun_out/s3i_ps.ncu-rep --page source --csv --print-source sass > gpurun_out/s3i_ps_src.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
