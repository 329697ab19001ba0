mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/s2e_tests.log 2>&1; tail -4 gpurun_out/s2e_tests.log
timeout 900 python bench.py > gpurun_out/s2e_bench.json 2> gpurun_out/s2e_bench.err; tail -c 300 gpurun_out/s2e_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/s2e_bench.json').read().strip().splitlines()[-1])
print(d['value'], d.get('rel_error'), d.get('selected_level'), {k:round(v['ms'],1) for k,v in d['stages_ms'].items()}, d['e2e']['value'], d.get('other_method',{}).get('ms_per_step'))"
