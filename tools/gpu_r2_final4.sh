# Round-2 closing evidence: GPU suite, smoke, default bench (all legs), config-1 latency
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2i_tests.log 2>&1; tail -3 gpurun_out/r2i_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2i_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2i_smoke.log
timeout 1200 python bench.py > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err; tail -c 300 gpurun_out/r2i_bench.err
for m in hpne pne; do timeout 300 python tools/latency_breakdown.py --method $m > gpurun_out/r2i_lat_$m.json 2> gpurun_out/r2i_lat_$m.err; done
timeout 300 python tools/latency_breakdown.py --method hpne --precision double > gpurun_out/r2i_lat_hpne_double.json 2>/dev/null
ls -la gpurun_out/r2i*
