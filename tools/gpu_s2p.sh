timeout 900 python -m pytest tests/test_gpu_qr_smem.py tests/test_gpu_qr16_golden.py tests/test_gpu_kernels.py -x -q > gpurun_out/s2p_tests.log 2>&1; tail -3 gpurun_out/s2p_tests.log
for lv in 16 32 64; do
  python tools/qr_probe.py 6144 2048 $lv
  SK_QR_SMEM=0 python tools/qr_probe.py 6144 2048 $lv
done > gpurun_out/s2p_qr.jsonl 2>&1
cat gpurun_out/s2p_qr.jsonl
