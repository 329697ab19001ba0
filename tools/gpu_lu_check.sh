# lu_smem_kernel check: bitwise vs lu_perm_kernel, the GPU suite, LU timings, one bench.
timeout 900 python -m pytest tests/test_gpu_lu_smem.py tests/test_gpu_kernels.py -x -q > gpurun_out/lu_tests.log 2>&1; echo rc=$? >> gpurun_out/lu_tests.log
(timeout 120 python tools/lu_probe.py 296 2048; SK_LU_KERNEL=perm timeout 120 python tools/lu_probe.py 296 2048) > gpurun_out/lu_probe.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu2.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_lu.json 2> gpurun_out/bench_lu.err
