set -x
timeout 600 python bench.py > gpurun_out/bench_v16.json 2> gpurun_out/bench_v16.err
tail -c 600 gpurun_out/bench_v16.json
timeout 600 ncu --set full --clock-control none -k regex:trsm_kernel --launch-skip 2 -c 1 -o gpurun_out/leaf4m -f python tools/trsm_oz_probe.py 4194304 2048 1 > gpurun_out/ncu_leaf.log 2>&1
timeout 600 ncu --set full --clock-control none -k 'regex:rowres|gemm_kernel|crt_sub' -c 3 -o gpurun_out/upd4m -f python tools/trsm_oz_probe.py 4194304 2048 1 > gpurun_out/ncu_upd.log 2>&1
python tools/ncu_summary.py gpurun_out/leaf4m.ncu-rep > gpurun_out/ncu_leaf.json 2>&1
python tools/ncu_summary.py gpurun_out/upd4m.ncu-rep > gpurun_out/ncu_upd.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_v16_1m.csv python bench.py --m 1048576 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
find gpurun_out -name "*.ncu-rep" -size +25M -delete
ls -la gpurun_out/
