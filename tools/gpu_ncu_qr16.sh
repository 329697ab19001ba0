# ncu --set full of the binary16 shared-memory level QR (the generator's binary64 flow kernel launches first)
B="python bench.py --m 1048576 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:householder_flow_kernel" --launch-skip 1 -c 1 \
    -o gpurun_out/ncu3_qr16 -f $B > gpurun_out/ncu3_qr16.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu3_qr16.ncu-rep > gpurun_out/ncu3_qr16.json 2>&1
ncu -i gpurun_out/ncu3_qr16.ncu-rep --page details --csv > gpurun_out/ncu3_qr16_details.csv 2>&1
find gpurun_out -name "*.ncu-rep" -size +25M -delete
