# Round-2 evidence: GPU suite, smoke, default bench (all legs), launch list at 1M rows,
# ncu --set full of the roofline kernel and of the round-2 kernels.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2f_tests.log 2>&1; tail -3 gpurun_out/r2f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2f_smoke.log; tail -2 gpurun_out/r2f_smoke.log
timeout 1200 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; tail -c 200 gpurun_out/r2f_bench.err
B="python bench.py --m 1048576 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/r2f_launches_1m.csv $B > gpurun_out/r2f_ncu_launch.log 2>&1
for k in trsm_kernel fft_pass_a fft_pass_b_tf32 jacobi_cta_kernel; do
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" -c 1 \
        -o gpurun_out/r2f_ncu_$k -f $B > gpurun_out/r2f_ncu_$k.log 2>&1
    python tools/ncu_summary.py gpurun_out/r2f_ncu_$k.ncu-rep > gpurun_out/r2f_ncu_$k.json 2>&1
done
find gpurun_out -name "*.ncu-rep" -size +25M -delete
ls -la gpurun_out/r2f*
