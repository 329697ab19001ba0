# QR index-arithmetic / guard-free fast paths: reference fixtures (bitwise), smem vs global, timings, GPU suite, bench.
timeout 900 python -m pytest tests/test_gpu_qr_smem.py tests/test_gpu_kernels.py tests/test_gpu_pipeline.py -x -q > gpurun_out/qr7_tests.log 2>&1; echo rc=$? >> gpurun_out/qr7_tests.log
(for lv in "6144 2048 16" "3000 1000 32" "6144 2048 32" "6144 2048 64"; do
   timeout 120 python tools/qr_probe.py $lv; SK_QR_SMEM=0 timeout 120 python tools/qr_probe.py $lv; done) > gpurun_out/qr7_probe.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu8.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu6.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_qr7.json 2> gpurun_out/bench_qr7.err
