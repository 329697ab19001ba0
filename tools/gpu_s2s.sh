timeout 600 ncu --set full --clock-control none --import-source on -k regex:householder_flow_kernel -c 1 -o gpurun_out/s2s_qr64 -f \
   python tools/qr_probe.py 6144 2048 64 > gpurun_out/s2s_qr64.log 2>&1
ncu -i gpurun_out/s2s_qr64.ncu-rep --page details --csv > gpurun_out/s2s_qr64_details.csv 2>/dev/null
ncu -i gpurun_out/s2s_qr64.ncu-rep --page source --csv --print-source sass > gpurun_out/s2s_qr64_src.csv 2>/dev/null
rm -f gpurun_out/s2s_qr64.ncu-rep
