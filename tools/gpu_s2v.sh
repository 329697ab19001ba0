timeout 1200 python -m pytest tests/test_gpu_qr_blocked.py tests/test_gpu_qr_smem.py -x -q > gpurun_out/s2v_tests.log 2>&1; tail -3 gpurun_out/s2v_tests.log
for lv in 32 64; do
  SK_QR_PROF=1 timeout 120 python tools/qr_probe.py 6144 2048 $lv 2>&1 | tail -2
  SK_QR_PANEL=flow SK_QR_PROF=1 timeout 120 python tools/qr_probe.py 6144 2048 $lv 2>&1 | tail -2
done
