for b in 1024 512; do
SK_TRSM_OZ_BASE=$b SK_TRSM_OZ_PROFILE=1 timeout 600 python tools/trsm_oz_probe.py 4194304 2048 3 > gpurun_out/s2m_$b.json 2> gpurun_out/s2m_$b.err
echo base=$b; grep ozaki gpurun_out/s2m_$b.json | head -2; grep trsm_ozaki gpurun_out/s2m_$b.err | tail -2
done
