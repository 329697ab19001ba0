timeout 1200 python -m pytest tests/test_gpu_qr_blocked.py tests/test_gpu_qr_smem.py tests/test_gpu_kernels.py tests/test_gpu_qr16_golden.py -x -q > gpurun_out/s2u_tests.log 2>&1; tail -25 gpurun_out/s2u_tests.log
for lv in 32 64; do
  timeout 120 python tools/qr_probe.py 6144 2048 $lv
  SK_QR_PANEL=flow timeout 120 python tools/qr_probe.py 6144 2048 $lv
  SK_QR_BLOCKED=0 timeout 120 python tools/qr_probe.py 6144 2048 $lv
done > gpurun_out/s2u_qr.jsonl 2>&1
cat gpurun_out/s2u_qr.jsonl
