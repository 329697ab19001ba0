# Round-2 session-2 check: FFT sketch parity + pass split, harness/CLI GPU tests, latency probe.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sketch_fft.py tests/test_harness_cli.py -m gpu -x -q > gpurun_out/s2a_tests.log 2>&1; tail -3 gpurun_out/s2a_tests.log
SK_FFT_PROFILE=1 timeout 600 python tools/bench_sketch.py --algos fft,tc > gpurun_out/s2a_sketch.json 2> gpurun_out/s2a_sketch.err
cat gpurun_out/s2a_sketch.json; grep 'sketch_fft M=' gpurun_out/s2a_sketch.err | sort | uniq -c | tail -8
timeout 300 python tools/latency_probe.py > gpurun_out/s2a_latency.jsonl 2>&1; tail -3 gpurun_out/s2a_latency.jsonl
