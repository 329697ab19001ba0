for b in 148 222 296 444 592 888 1184; do timeout 120 python tools/lu_probe.py $b 2048; done > gpurun_out/lu_sweep.txt 2>&1
