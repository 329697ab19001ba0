timeout 900 python -m pytest tests/test_gpu_qr_blocked.py tests/test_gpu_qr_smem.py -x -q 2>&1 | tail -2
for lv in 32 64; do timeout 120 python tools/qr_probe.py 6144 2048 $lv; SK_QR_PROF=1 timeout 120 python tools/qr_probe.py 6144 2048 $lv 2>&1 | grep blocked | tail -1; done
