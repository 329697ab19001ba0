mkdir -p gpurun_out
for cl16 in 0 1024 3000; do for lv in 32 64; do SK_QR_CL16_ROWS=$cl16 timeout 300 python tools/qr_probe.py 6144 2048 $lv 2>&1 | tail -1 | sed "s/^/cl16=$cl16 /" >> gpurun_out/s3v_qr.txt; done; done
for cl16 in 0 1024; do SK_QR_CL16_ROWS=$cl16 timeout 300 python tools/qr_probe.py 3000 1000 32 2>&1 | tail -1 | sed "s/^/cl16=$cl16 /" >> gpurun_out/s3v_qr.txt; done
