mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_round2.py tests/test_gpu_pipeline.py -x -q > gpurun_out/s2n_tests.log 2>&1; tail -3 gpurun_out/s2n_tests.log
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/s2n_bench.json 2> gpurun_out/s2n_bench.err; tail -c 300 gpurun_out/s2n_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/s2n_bench.json').read().strip().splitlines()[-1])
print(d['value'], {k:round(v['ms'],1) for k,v in d['stages_ms'].items()}, d['e2e']['value'], d['e2e'].get('pageable_numpy'), d.get('clocks'))"
