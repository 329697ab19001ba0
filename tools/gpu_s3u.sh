mkdir -p gpurun_out
for cl4 in 0 3072; do for lv in 32 64; do SK_QR_CL4_ROWS=$cl4 timeout 300 python tools/qr_probe.py 3000 1000 $lv | sed "s/^/cl4=$cl4 /" >> gpurun_out/s3u_qr.txt 2>&1; done; done
for cl4 in 0 6144; do SK_QR_CL4_ROWS=$cl4 timeout 300 python tools/qr_probe.py 6144 2048 32 | sed "s/^/cl4=$cl4 /" >> gpurun_out/s3u_qr.txt 2>&1; done
