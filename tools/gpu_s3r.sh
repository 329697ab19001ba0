mkdir -p gpurun_out
python tools/sketch_dmma_probe.py 100000 1000 > gpurun_out/s3r_probe.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sketch_kernel -c 1 -o gpurun_out/s3r_sk -f python tools/sketch_dmma_probe.py 100000 1000 > gpurun_out/s3r_ncu.log 2>&1
ncu -i gpurun_out/s3r_sk.ncu-rep --page details --csv > gpurun_out/s3r_details.csv 2>/dev/null
ncu -i gpurun_out/s3r_sk.ncu-rep --page source --csv --print-source sass > gpurun_out/s3r_src.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
