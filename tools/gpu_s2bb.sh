timeout 300 python -m pytest tests/test_gpu_trsm_ozaki.py -x -q > gpurun_out/s2bb_tests.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/s2bb_tests.log
for mc in 1 0; do SK_OZ_MC=$mc SK_TRSM_OZ_PROFILE=1 timeout 300 python tools/trsm_oz_probe.py 4194304 2048 2 2>&1 | grep -E '"ozaki"|trsm_ozaki' | tail -2 | sed "s/^/mc=$mc /"; done
