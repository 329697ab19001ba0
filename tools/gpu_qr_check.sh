# smem-resident level QR check: bitwise vs the global flow kernel, QR timings, GPU suite, bench.
timeout 900 python -m pytest tests/test_gpu_qr_smem.py -x -q > gpurun_out/qr_tests.log 2>&1; echo rc=$? >> gpurun_out/qr_tests.log
(for lv in "6144 2048 16" "6144 2048 32" "3000 1000 32" "6144 2048 64"; do
   timeout 120 python tools/qr_probe.py $lv; SK_QR_SMEM=0 timeout 120 python tools/qr_probe.py $lv; done) > gpurun_out/qr_probe.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu3.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_qr.json 2> gpurun_out/bench_qr.err
