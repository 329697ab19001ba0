# Round-1 closing evidence on the final build: config-3 kappa points (binary32 / binary64
# levels), the PNE leg, the launch list at 1M rows and one `ncu --set full` capture of each
# kernel not yet covered by profiles/ (tcgen05 sketch, its prep pass, level QR, LU, Hager,
# Cholesky, residual).  Run from the repo root under gpurun.
set -x
B="python bench.py --m 1048576 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 python bench.py --kappa 1e3 --no-cpu-baseline --no-e2e > gpurun_out/bench_k1e3.json 2> gpurun_out/bench_k1e3.err
timeout 900 python bench.py --kappa 2e6 --no-cpu-baseline --no-e2e > gpurun_out/bench_k2e6.json 2> gpurun_out/bench_k2e6.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/launches_r1_final_1m.csv $B > gpurun_out/ncu_launch.log 2>&1
for k in sketch_tc_kernel prep_f16r householder_flow_kernel lu_perm_kernel hager_kernel chol_blocked_kernel residual_kernel; do
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" -c 1 \
        -o gpurun_out/ncu_$k -f $B > gpurun_out/ncu_$k.log 2>&1
    python tools/ncu_summary.py gpurun_out/ncu_$k.ncu-rep > gpurun_out/ncu_$k.json 2>&1
done
find gpurun_out -name "*.ncu-rep" -size +25M -delete
ls -la gpurun_out/
