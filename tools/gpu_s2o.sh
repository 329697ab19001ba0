timeout 900 python -m pytest tests/test_gpu_jacobi.py tests/test_gpu_kernels.py -x -q > gpurun_out/s2o_tests.log 2>&1; tail -3 gpurun_out/s2o_tests.log
timeout 900 python tools/diag_cost.py > gpurun_out/s2o_diag.json 2> gpurun_out/s2o_diag.err; cat gpurun_out/s2o_diag.json
