mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_trsm_ozaki.py tests/test_gpu_round2.py -x -q > gpurun_out/s2j_tests.log 2>&1; tail -3 gpurun_out/s2j_tests.log
SK_TRSM_OZ_PROFILE=1 timeout 600 python tools/trsm_oz_probe.py > gpurun_out/s2j_trsm.json 2> gpurun_out/s2j_trsm.err
cat gpurun_out/s2j_trsm.json; grep trsm_ozaki gpurun_out/s2j_trsm.err | tail -3
