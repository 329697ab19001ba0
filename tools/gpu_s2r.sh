for k in 1e3 2e6; do
  timeout 900 python bench.py --kappa $k --no-e2e --no-cpu-baseline > gpurun_out/s2r_k$k.json 2> gpurun_out/s2r_k$k.err
  python -c "
import json; d=json.loads(open('gpurun_out/s2r_k$k.json').read().strip().splitlines()[-1])
print('$k', d['value'], d.get('selected_level'), d.get('rel_error'), {k:round(v['ms'],1) for k,v in d['stages_ms'].items()}, d.get('other_method',{}).get('ms_per_step'), d.get('clocks',{}).get('sm_mhz'))"
done
