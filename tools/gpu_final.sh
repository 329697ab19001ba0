# Final round-1 evidence: GPU suite, smoke, bench (all legs), ncu of the main kernels.
set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
tail -c 400 gpurun_out/bench_final.json
timeout 600 ncu --set full --clock-control none -k 'regex:gemm_kernel|residues_kernel|sketch_tc_kernel|residual_kernel|colstats_kernel' -c 6 -o gpurun_out/kern1m -f python bench.py --m 1048576 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_kern.log 2>&1
python tools/ncu_summary.py gpurun_out/kern1m.ncu-rep > gpurun_out/ncu_kern.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_final_1m.csv python bench.py --m 1048576 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_final.log 2>&1
find gpurun_out -name "*.ncu-rep" -size +25M -delete
ls -la gpurun_out/
