# Final evidence for the round-1 build with the shared-memory LU / QR: full default bench,
# smoke, launch list and ncu of the two new kernels.
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo rc=$? >> gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err
B="python bench.py --m 1048576 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/launches_r1_final2_1m.csv $B > gpurun_out/ncu_launch2.log 2>&1
for k in lu_smem_kernel householder_flow_kernel; do
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" -c 1 \
        -o gpurun_out/ncu2_$k -f $B > gpurun_out/ncu2_$k.log 2>&1
    python tools/ncu_summary.py gpurun_out/ncu2_$k.ncu-rep > gpurun_out/ncu2_$k.json 2>&1
done
find gpurun_out -name "*.ncu-rep" -size +25M -delete
