mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_lu_smem.py tests/test_gpu_qr_blocked.py -x -q > gpurun_out/s3o_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3o_tests.log
