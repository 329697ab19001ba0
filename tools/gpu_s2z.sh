timeout 600 ncu --set full --clock-control none --import-source on -k regex:qrb_panel_cluster -c 1 -o gpurun_out/s2z_pc -f \
   python tools/qr_probe.py 6144 2048 32 > gpurun_out/s2z.log 2>&1
ncu -i gpurun_out/s2z_pc.ncu-rep --page details --csv > gpurun_out/s2z_details.csv 2>/dev/null
ncu -i gpurun_out/s2z_pc.ncu-rep --page source --csv --print-source sass > gpurun_out/s2z_src.csv 2>/dev/null
rm -f gpurun_out/s2z_pc.ncu-rep
