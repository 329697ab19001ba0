mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py -k "full_size" -x -q > gpurun_out/s2k_c2.log 2>&1; tail -3 gpurun_out/s2k_c2.log
timeout 900 python -m pytest tests/test_harness_cli.py -m gpu -x -q > gpurun_out/s2k_h.log 2>&1; tail -3 gpurun_out/s2k_h.log
timeout 900 python tools/config5_parity.py --m 65536 --n 256 --kappas 1e2,1e10 --rhos 1e-10,1e-2 > gpurun_out/s2k_c5small.jsonl 2> gpurun_out/s2k_c5small.err
tail -c 1500 gpurun_out/s2k_c5small.jsonl; tail -5 gpurun_out/s2k_c5small.err
