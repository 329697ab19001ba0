timeout 1500 python -m pytest tests/test_gpu_qr_blocked.py tests/test_gpu_qr_smem.py tests/test_gpu_kernels.py tests/test_gpu_pipeline.py -x -q > gpurun_out/s2aa_tests.log 2>&1; tail -3 gpurun_out/s2aa_tests.log
for lv in 32 64; do timeout 120 python tools/qr_probe.py 6144 2048 $lv; SK_QR_LOOKAHEAD=0 timeout 120 python tools/qr_probe.py 6144 2048 $lv; done
